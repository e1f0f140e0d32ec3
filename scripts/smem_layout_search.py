"""Search shared-memory row/plane padding (R, P) per order for the pencil
kernels: minimise modeled wavefronts of the three pencil access orientations
(8-byte accesses, half-warp = 16 lanes, 16 eight-byte bank pairs; identical
addresses broadcast).  Prints the best (R, P) per NQ."""
import itertools
import sys

EPB = {2: 32, 3: 14, 4: 4, 5: 5, 6: 2, 7: 2, 8: 1, 9: 1, 10: 1, 11: 1, 12: 1, 13: 1, 14: 1,
       15: 1, 16: 1}


def cost(NQ, R, P, swz=None):
    VOL = NQ * P
    T = EPB[NQ] * NQ * NQ
    tot = 0
    for orient in range(3):
        for m in range(NQ):
            for w0 in range(0, T, 32):
                for h0 in (w0, w0 + 16):
                    banks = {}
                    for t in range(h0, min(h0 + 16, T)):
                        le, tt = divmod(t, NQ * NQ)
                        a, b = tt % NQ, tt // NQ
                        if orient == 0:
                            k, j, i = b, a, m
                        elif orient == 1:
                            k, j, i = b, m, a
                        else:
                            k, j, i = m, b, a
                        addr = le * 3 * VOL + k * P + j * R + (i if swz is None else swz(k, j, i))
                        banks.setdefault(addr % 16, set()).add(addr)
                    tot += max((len(v) for v in banks.values()), default=0)
    return tot


def ideal(NQ):
    T = EPB[NQ] * NQ * NQ
    n_half = sum(1 for w0 in range(0, T, 32) for h0 in (w0, w0 + 16) if h0 < T)
    return 3 * NQ * n_half


if __name__ == "__main__":
    for NQ in range(2, 17):
        base = (NQ if NQ % 2 else NQ + 1, None)
        best = None
        for R in range(NQ, NQ + 4):
            for P in range(NQ * R, NQ * R + 9):
                c = cost(NQ, R, P)
                if best is None or c < best[0] or (c == best[0] and R * P < best[1] * best[2]):
                    best = (c, R, P)
        Rc = NQ if NQ % 2 else NQ + 1
        Pc = NQ * Rc + (1 if (NQ * Rc) % 2 == 0 else 0)
        cur = cost(NQ, Rc, Pc)
        print(f"NQ={NQ:2d} ideal={ideal(NQ):5d} current(R={Rc},P={Pc})={cur:5d} "
              f"best(R={best[1]},P={best[2]})={best[0]:5d}")
        sys.stdout.flush()


def search_rot(NQ):
    best = None
    for R in range(NQ, NQ + 3):
        for P in range(NQ * R, NQ * R + 5):
            for c1 in range(NQ):
                for c2 in range(NQ):
                    swz = (lambda k, j, i, c1=c1, c2=c2: (i + c1 * j + c2 * k) % NQ)
                    c = cost(NQ, R, P, swz)
                    key = (c, R * P)
                    if best is None or key < best[0]:
                        best = (key, R, P, c1, c2)
    return best
