"""Element partitioning -- ``nekmini.partition.rcb``.

Recursive coordinate bisection on the host (setup): split each subset at the
median along its longest bounding-box axis (lowest axis on ties), ordering
by (coordinate, element index); P_lo = P // 2 ranks take floor(n P_lo / P)
elements, so part sizes differ by at most one.  For a box of
nx x ny x nz elements and P = 2^k this yields contiguous brick blocks.
"""

import numpy as np

__all__ = ["rcb", "rank_elements"]


def rcb(centroids, P):
    pts = np.asarray(centroids, dtype=np.float64)
    out = np.empty(len(pts), dtype=np.int64)
    stack = [(np.arange(len(pts)), 0, int(P))]
    while stack:
        idx, first, nparts = stack.pop()
        if nparts <= 1 or len(idx) == 0:
            out[idx] = first
            continue
        sub = pts[idx]
        axis = int(np.argmax(sub.max(axis=0) - sub.min(axis=0)))
        srt = idx[np.lexsort((idx, sub[:, axis]))]
        lo_parts = nparts // 2
        cut = len(idx) * lo_parts // nparts
        stack.append((srt[cut:], first + lo_parts, nparts - lo_parts))
        stack.append((srt[:cut], first, lo_parts))
    return out


def rank_elements(part, rank):
    """Global element indices owned by `rank`, ascending."""
    return np.flatnonzero(np.asarray(part) == rank)
