"""Partition-efficiency (Fig. 4) and ghost-children ratio (Fig. 5,
P:836-860) sweeps over the paper's mesh sequences, computed by the library's
exact integer partition model.  Writes a CSV (the figures' data; plots are out
of scope).

    python tools/sweeps.py [out.csv]
"""
import csv
import sys
import time
from fractions import Fraction

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1904_03317_b200 as G  # noqa: E402

SWEEP = {
    2: {"uniform": range(8, 13), "circle": range(10, 17), "quadrant": range(8, 14), "annulus": range(8, 14)},
    3: {"uniform": range(4, 8), "circle": range(6, 11), "quadrant": range(5, 9), "annulus": range(5, 9)},
}
PS = {2: (4, 16, 64, 256, 1024, 2048, 4096, 8192, 16384), 3: (8, 64, 512, 4096)}


def main(out):
    rows = []
    t0 = time.time()
    for d, kinds in SWEEP.items():
        for kind, Ls in kinds.items():
            for L in Ls:
                f = G.gmg_forest_sequence(d, kind, L)
                n = f.info()["n_leaves"]
                for p in PS[d]:
                    if p > n:
                        continue
                    m = G.gmg_partition(f, p).model()
                    eta = Fraction(*m["eta"])
                    gc, ch = sum(m["ghost_children"]), sum(m["children"])
                    rows.append(dict(kind=kind, dim=d, L=L, n_leaves=n, p=p, leaves_per_rank=n / p,
                                     eta=float(eta), eta_exact=f"{eta.numerator}/{eta.denominator}",
                                     W_opt=float(Fraction(*m["W_opt"])), W_sync=m["W_sync"], W=m["W"],
                                     ghost_children=gc, children=ch, ghost_ratio=gc / max(ch, 1)))
                print(f"{kind:8s} d={d} L={L:2d} leaves={n:9d} {time.time() - t0:6.1f}s", flush=True)
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_fig4_fig5_sweeps.csv")
