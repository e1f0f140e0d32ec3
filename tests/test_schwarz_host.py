"""CPU: host-side Schwarz setup of the product (face-neighbour map, batched
1-D FDM eigenproblems) against oracle/schwarz.py -- integer maps bit-exact,
1-D operators to 1e-12."""

import numpy as np
import pytest

from oracle import mesh as om
from oracle import schwarz as osz
from paper_2104_05829_b200 import schwarz as sz
from paper_2104_05829_b200.basis import SpectralBasis

CODES = {"nbr": 0, "neu": 1, "dir": 2}


@pytest.mark.parametrize("counts,N,bc", [((3, 2, 2), 3, "dirichlet"), ((2, 1, 3), 4, "periodic"),
                                          ((1, 1, 1), 5, "periodic"), ((2, 2, 1), 2, "neumann"),
                                          ((3, 3, 3), 7, {"x-": "periodic", "x+": "periodic",
                                                          "y-": "dirichlet", "z+": "dirichlet"})])
def test_face_map_matches_oracle(counts, N, bc):
    m = om.build_box_mesh((1, 1, 1), counts, N, bc=bc, deformation=None)
    a = sz.face_source_map(m.ids, m.E, N)
    b = osz.face_source_map(m.ids, m.E, N)
    assert np.array_equal(a, b)


def test_face_map_shuffled_element_order():
    """Neighbours follow the ids, not the element order (HEXMESH meshes)."""
    N = 3
    m = om.build_box_mesh((1, 1, 1), (3, 2, 2), N, bc="dirichlet")
    nq = N + 1
    perm = np.random.default_rng(4).permutation(m.E)
    ids = m.ids.reshape(m.E, -1)[perm].ravel()
    f = sz.face_source_map(ids, m.E, N)
    f0 = osz.face_source_map(m.ids, m.E, N)
    inv = np.argsort(perm)
    # map local indices of the shuffled layout back to the original layout
    loc_new_to_old = (perm[:, None] * nq ** 3 + np.arange(nq ** 3)[None, :]).ravel()
    back = np.where(f >= 0, loc_new_to_old[np.maximum(f, 0)], -1)
    assert np.array_equal(back[inv], f0)


@pytest.mark.parametrize("N", [1, 2, 3, 7, 15])
def test_fdm_1d_batch_matches_oracle(N):
    b = SpectralBasis.get(N)
    kinds = ["nbr", "neu", "dir"]
    pairs = [(l, r) for l in kinds for r in kinds]
    h = np.linspace(0.3, 1.7, len(pairs))
    S, lam = sz.fdm_1d_batch(b.diff, b.weights, h, np.array([CODES[l] for l, _ in pairs]),
                             np.array([CODES[r] for _, r in pairs]))
    S, lam = S.numpy(), lam.numpy()
    for q, (l, r) in enumerate(pairs):
        So, lo, keep = osz.fdm_1d(b.diff, b.weights, h[q], l, r)
        f = lambda L: np.where(np.isfinite(L), 1.0 / (np.where(np.isfinite(L), L, 0) + 1.0), 0)
        P = S[q] @ np.diag(f(lam[q])) @ S[q].T
        Po = So @ np.diag(f(lo)) @ So.T
        assert np.max(np.abs(P - Po)) < 1e-12 * max(1.0, np.max(np.abs(Po)))
        assert np.sum(np.isfinite(lam[q])) == keep.sum()
        assert np.allclose(np.sort(lam[q][np.isfinite(lam[q])]), np.sort(lo[:keep.sum()]), rtol=1e-10, atol=1e-10)
