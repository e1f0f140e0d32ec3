"""The compiled CPU oracle (oracle/c/bk5_cpu.c) against the numpy oracle:
the bench's CPU baseline / reference arm computes the same operator."""

import numpy as np
import pytest

from oracle import cpu_bk5
from oracle import mesh as om
from oracle import operators as oop


@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 9, 12, 15])
def test_cpu_bk5_matches_numpy_oracle(N):
    o = om.build_box_mesh((1.0, 1.0, 1.0), (3, 2, 2), N, deformation=("sine", 0.05))
    rng = np.random.default_rng(N)
    u = rng.standard_normal((o.E, N + 1, N + 1, N + 1))
    ref = oop.bk5(o.basis.diff, o.G, u)
    w, used = cpu_bk5.bk5(o.basis.diff, o.G, u)
    assert used >= 1
    assert np.linalg.norm(w - ref) / np.linalg.norm(ref) < 1e-13
    lam0, lam1 = 0.3, 2.0
    ref = oop.bk5(o.basis.diff, o.G, u, lam0=lam0, B=o.B, lam1=lam1)
    w, _ = cpu_bk5.bk5(o.basis.diff, o.G, u, lam0=lam0, B=o.B, lam1=lam1, threads=1)
    assert np.linalg.norm(w - ref) / np.linalg.norm(ref) < 1e-13


def test_cpu_bk5_thread_count_invariant():
    o = om.build_box_mesh((1.0, 1.0, 1.0), (4, 3, 2), 7, deformation=("sine", 0.05))
    u = np.random.default_rng(0).standard_normal((o.E, 8, 8, 8))
    w1, _ = cpu_bk5.bk5(o.basis.diff, o.G, u, threads=1)
    w4, used = cpu_bk5.bk5(o.basis.diff, o.G, u, threads=4)
    assert used == 4 and np.array_equal(w1, w4)   # element-parallel: same bits
