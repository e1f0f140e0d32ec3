"""CPU oracle for the SEM Poisson hot path (TEST INFRASTRUCTURE ONLY).

This package is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import it.  The product package
(``paper_2104_05829_b200``) never imports anything from here and fails loudly
when its CUDA library is missing.

What it restates, and how each part is pinned:

* ``oracle.basis``     -- GLL nodes/weights/D-hat, restating
  /root/reference/pkg/src/nekmini/basis.py:18-96.  PINNED: checked bit-for-bit
  against golden vectors produced by the reference module itself
  (tests/golden/make_golden.py -> tests/golden/basis_ref.npz) and against the
  reference's own test cases (test_basis.py:12-129, restated in
  tests/test_oracle_basis.py).
* ``oracle.mesh``      -- box meshes, geometric factors, global ids, masks,
  HEXMESH v1.  No reference code exists for these; pinned to
  the SPEC known-answer examples.
* ``oracle.gs``        -- gs_setup / gs_op in canonical order.
  Pinned to SPEC examples and to an explicit dense 0/1 Q-matrix oracle.
* ``oracle.operators`` -- BK5 stiffness, mass, Jacobi diagonal
  (SPEC.md:370-408).  Pinned to a dense element matrix
  assembled from Eq. (25) by quadrature (independent of sum factorisation).
* ``oracle.solvers``   -- PCG / flexible PCG.  Pinned to SPEC
  examples and a dense direct solve.
* ``oracle.partition`` -- RCB.  Pinned to SPEC examples.

The reference ships no implementation of Ax, gs or CG, so for
those the parity anchor is the SPEC contract plus the dense oracles above, not
reference-generated vectors.  See DESIGN.md "Parity and the oracle".
"""
