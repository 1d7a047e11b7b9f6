"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    out = []
    for r in rows[hi + 1:]:
        v = float(r[h.index("Metric Value")].replace(",", ""))
        u = r[h.index("Metric Unit")]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        out.append((r[h.index("Kernel Name")].split("(")[0].replace("void gmg::dev::", ""), r[h.index("Grid Size")], v))
    return out


if __name__ == "__main__":
    L = load(sys.argv[1])
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    T = sum(v for _, _, v in L)
    for n, g, v in L:
        tot[n] += v
        cnt[n] += 1
    print(f"total {T:.1f} us over {len(L)} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.1f} us {100 * v / T:5.1f}%  n={cnt[k]:3d}  {k}")
    if len(sys.argv) > 2:
        for n, g, v in L[: int(sys.argv[2])]:
            print(f"{v:9.1f} {g:>16s} {n}")
