"""Quick A/B timing of the V-cycle kernels on one config (no bench line): V-cycle
time (CUDA events, graph) and the top kernels of gmg_profile_vcycle.  Knobs are
environment variables read at setup (GMG_GFAM, GMG_GF_SLOTS, GMG_FUSE_PROLONG)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, config_c5, uniform_pm1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--mixed", action="store_true")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--tag", default="")
args = ap.parse_args()
cfg = config_c5(1) if args.config == "c5" else config(args.config)
coef = None
if cfg.get("coef") == "level2_log_uniform":          # config 4: a per level-2 cell
    from gmg_inputs import log_uniform_coef
    coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
_, _, h = G.build_config(cfg, mixed=args.mixed, coef_level2=coef)
info = h.info()
b = torch.tensor(uniform_pm1(info["n_leaf_free"]), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
for _ in range(5):
    h.vcycle(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(args.steps):
    h.vcycle(b, x)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / args.steps
recs = h.profile_vcycle(b, x, n_rep=2)
recs = [r for r in recs if r["launches"]]
recs.sort(key=lambda r: -r["seconds"])
top = [(r["kind"], r["level"], round(1e6 * r["seconds"] / r["launches"], 1), round(r["seconds"] / 2 / ms * 1e3, 3))
       for r in recs[:10]]
per_level = {}
for r in recs:
    per_level[r["level"]] = per_level.get(r["level"], 0.0) + r["seconds"] / 2
launches = {}
for r in recs:
    launches[r["level"]] = launches.get(r["level"], 0) + r["launches"] // 2
print(json.dumps({"tag": args.tag, "config": args.config, "ms": ms, "dofs_per_s": info["n_leaf_nodes"] / ms * 1e3,
                  "gf": sum(info["level_gf"]), "top": top,
                  "per_level_us": {l: round(1e6 * v, 1) for l, v in sorted(per_level.items())},
                  "per_level_launch_records": launches}))
