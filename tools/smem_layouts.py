"""Search the shared-memory transposition layouts of fam_tensor_apply (Q2 3D).

A block of 4 warps runs 5 families, thread t = 25 s + line (s = family slot,
line = c0 + 5 c1 over the two coordinates a pass keeps fixed per lane; threads
125..127 idle), so warps straddle two families.  A layout maps patch node
(x, y, z), 0 <= x, y, z < 5, of slot s to s S + cx x + cy y + cz z.  Wavefront
model: fp64 accesses are served per 16-lane half-warp over 16 bank pairs, fp32
accesses in one pass over 32 banks; the cost of an access is the maximum number
of distinct words on one bank (pair).  For every slot stride S prints
the minimal layouts A (z-pass store / y-pass load), B (y-pass store / x-pass
load) and N (x-pass store / z-line scatter load); then the costs of the choice
kernels.cuh:PatchLayout makes (A, B and N each with its own slot stride).  A
and B reach the ideal with a slot stride S = 25 (mod 16 resp. 32) and
coefficients (a, 5a, 5a) resp. (a, a, 5a) mod the bank count; N cannot (the
roles of y in the two line numberings differ, an odd cycle), its best is
printed.  Ideal per pass and array (5 q x 4 warps): 40 fp64, 20 fp32 wavefronts.
"""
import itertools
from collections import Counter

R = range(5)


def wf64(addrs):
    t = 0
    for h in (addrs[:16], addrs[16:]):
        h = [a for a in h if a is not None]
        if h:
            t += max(Counter(v % 16 for v in set(h)).values())
    return t


def wf32(addrs):
    h = [a for a in addrs if a is not None]
    return max(Counter(v % 32 for v in set(h)).values()) if h else 0


def cost(wf, L, S, kind):
    cx, cy, cz = L
    f = lambda x, y, z: cx * x + cy * y + cz * z
    tot = 0
    for q in R:
        for w in range(4):
            addrs = []
            for lane in range(32):
                t = 32 * w + lane
                if t >= 125:
                    addrs.append(None)
                    continue
                s, line = divmod(t, 25)
                c0, c1 = line % 5, line // 5
                a = {"z": f(c0, c1, q), "y": f(c0, q, c1), "x": f(q, c0, c1)}[kind]
                addrs.append(s * S + a)
            tot += wf(addrs)
    return tot


lays = []
for cx, cy, cz in itertools.product(range(1, 40), repeat=3):
    idx = [cx * x + cy * y + cz * z for x in R for y in R for z in R]
    if len(set(idx)) == 125 and max(idx) <= 180:
        lays.append(((cx, cy, cz), max(idx) + 1))

for name, wf, banks in (("fp64", wf64, 16), ("fp32", wf32, 32)):
    for S in range(125, 125 + banks):   # slot stride (slots must not overlap: layout size <= S)
        res = [(L, sz, cost(wf, L, S, "z"), cost(wf, L, S, "y"), cost(wf, L, S, "x")) for L, sz in lays if sz <= S]
        A = min(res, key=lambda r: (r[2] + r[3], r[1]))
        B = min(res, key=lambda r: (r[3] + r[4], r[1]))
        N = min(res, key=lambda r: (r[4] + r[2], r[1]))
        print(f"{name} S={S:3d}  A {A}  B {B}  N {N}   (layout, size, z, y, x)")

print("kernels.cuh choice (wavefronts per pass and array, 5 families):")
for name, wf, A, B, N, SAB, SN in (("fp64", wf64, (1, 5, 37), (1, 33, 5), (1, 5, 25), 185, 125),
                                   ("fp32", wf32, (1, 5, 37), (1, 33, 5), (1, 5, 39), 185, 185)):
    print(f"  {name}: A {A} S={SAB}: z-store {cost(wf, A, SAB, 'z')} y-load {cost(wf, A, SAB, 'y')}; "
          f"B {B} S={SAB}: y-store {cost(wf, B, SAB, 'y')} x-load {cost(wf, B, SAB, 'x')}; "
          f"N {N} S={SN}: x-store {cost(wf, N, SN, 'x')} z-load {cost(wf, N, SN, 'z')}")
