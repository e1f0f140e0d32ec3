"""Oracle: recursive coordinate bisection.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates SPEC.md:286-294: recursive median split along the longest axis of
each subset's bounding box; ties in the sort broken by (coordinate, element
index); ties in axis length broken by lowest axis; P not a power of two split
as P_lo = P // 2 ranks receiving floor(n * P_lo / P) elements; balance
max - min <= 1.
"""

import numpy as np


def rcb(centroids, P):
    c = np.asarray(centroids, dtype=np.float64)
    n = c.shape[0]
    part = np.zeros(n, dtype=np.int64)

    def rec(idx, r0, p):
        if p == 1 or len(idx) == 0:
            part[idx] = r0
            return
        pts = c[idx]
        ext = pts.max(axis=0) - pts.min(axis=0)
        ax = int(np.argmax(ext))
        order = np.lexsort((idx, pts[:, ax]))
        plo = p // 2
        nlo = (len(idx) * plo) // p
        rec(idx[order[:nlo]], r0, plo)
        rec(idx[order[nlo:]], r0 + plo, p - plo)

    rec(np.arange(n), 0, int(P))
    return part
