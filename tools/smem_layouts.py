"""Search the shared-memory transposition layouts of fam_tensor_apply (Q2 3D).

A layout maps patch node (x, y, z), 0 <= x, y, z < 5, to cx x + cy y + cz z.
Lanes are numbered c0 + 5 c1 over the two coordinates a pass keeps fixed per
lane.  Wavefront model: fp64 accesses are served per 16-lane half-warp over 16
bank pairs, fp32 accesses in one pass over 32 banks; the cost of an access is
the maximum number of distinct words on one bank (pair).  Prints the minimal
layouts A (z-pass store / y-pass load) and B (y-pass store / x-pass load) that
kernels.cuh:PatchLayout uses.
"""
import itertools
from collections import Counter

R = range(5)


def wf64(a):
    f = lambda h: max(Counter(v % 16 for v in h).values()) if h else 0
    return f(a[:16]) + f(a[16:])


def wf32(a):
    return max(Counter(v % 32 for v in a).values())


def lanes(fn, fixed):
    return [fn(c0, c1, fixed) for c1 in R for c0 in R]


for name, wf in (("fp64", wf64), ("fp32", wf32)):
    res = []
    for cx, cy, cz in itertools.product(range(1, 40), repeat=3):
        idx = [cx * x + cy * y + cz * z for x in R for y in R for z in R]
        if len(set(idx)) < 125 or max(idx) > 180:
            continue
        L = lambda x, y, z: cx * x + cy * y + cz * z
        zs = max(wf(lanes(lambda px, py, z: L(px, py, z), z)) for z in R)
        yl = max(wf(lanes(lambda px, pz, q: L(px, q, pz), q)) for q in R)
        xl = max(wf(lanes(lambda py, pz, q: L(q, py, pz), q)) for q in R)
        res.append(((cx, cy, cz), max(idx) + 1, zs, yl, xl))
    A = min(res, key=lambda r: (r[2] + r[3], r[1]))
    B = min(res, key=lambda r: (r[3] + r[4], r[1]))
    nat = [r for r in res if r[0] == (1, 5, 25)][0]
    print(f"{name}: natural {nat}  A {A}  B {B}   (layout, size, z-store, y-access, x-access)")
