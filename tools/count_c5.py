"""Exact sizes of the config-5 weak-scaling forests (reading R21): the smallest
shell half-width w = m 2^-10 whose forest has >= 125M n leaf nodes, for n = 1,
2, 4, 8 (library forest generator + gmg_forest_count_nodes; CPU only).  Writes
profiles/c5_shell_counts.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import CONFIGS  # noqa: E402

OUT = os.path.join(ROOT, "profiles", "c5_shell_counts.json")
counts = json.load(open(OUT)) if os.path.exists(OUT) else {}


def count(m):
    key = str(m)
    if key in counts:
        return counts[key]["nodes"]
    cfg = dict(CONFIGS["c5"])
    cfg["shell"] = (m, 1024)
    t = time.time()
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    n = f.count_nodes(cfg["k"])
    leaves = f.info()["n_leaves"]
    del f
    counts[key] = {"nodes": n, "leaves": leaves, "seconds": round(time.time() - t, 1)}
    json.dump(counts, open(OUT, "w"), indent=1, sort_keys=True)
    print(f"m={m}: {n} nodes, {leaves} leaves ({time.time() - t:.0f} s)", flush=True)
    return n


result = {}
for n_gpus, guess in ((1, 4), (2, 11), (4, 24), (8, 50)):
    target = 125_000_000 * n_gpus
    m = guess
    while count(m) < target:
        m += 1
    while m > 0 and count(m - 1) >= target:
        m -= 1
    result[n_gpus] = m
    print(f"n={n_gpus}: m={m}", flush=True)
counts["smallest_m"] = {str(k): v for k, v in result.items()}
json.dump(counts, open(OUT, "w"), indent=1, sort_keys=True)
