"""Oracle: compiled CPU BK5 (oracle/c/bk5_cpu.c, C + OpenMP).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The same operator as
``oracle.operators.bk5``, compiled so
that the bench's CPU baseline and ``--impl reference`` arm time a CPU path
no Python process pool can beat (VERDICT r1 "What's weak" 4).  Pinned to the
numpy oracle in tests/test_oracle_cpu_bk5.py (1e-13 relative L2).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "c", "libbk5cpu.so")
_lib = None


def build():
    subprocess.run(["make", "-C", os.path.join(_HERE, "c")], check=True,
                   stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        L.bk5_cpu.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4 + \
            [ctypes.c_double, ctypes.c_void_p, ctypes.c_double, ctypes.c_int]
        L.bk5_cpu.restype = ctypes.c_int
        _lib = L
    return _lib


def bk5(D, G, u, lam0=1.0, B=None, lam1=0.0, out=None, threads=0):
    """w = lam0 A_L u + lam1 B u; threads <= 0: all (OpenMP default).
    Returns (w, threads_used)."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    E, nq = u.shape[0], u.shape[1]
    w = np.empty_like(u) if out is None else out
    Bp = None if B is None else np.ascontiguousarray(B, dtype=np.float64)
    used = lib().bk5_cpu(nq - 1, E, D.ctypes.data, G.ctypes.data, u.ctypes.data, w.ctypes.data,
                         float(lam0), None if Bp is None else Bp.ctypes.data, float(lam1),
                         int(threads))
    if used < 0:
        raise ValueError("bk5_cpu: invalid arguments")
    return w, used
