"""Driver for ncu captures of the V-cycle kernels: builds a config (gmg_inputs
name, optional c5 n), runs warm-up V-cycles, then one V-cycle between
cudaProfilerStart/Stop.  Use with ncu --profile-from-start off, e.g.

  ncu --profile-from-start off --set full --clock-control none --import-source on \\
      -k regex:gfam_tensor_apply --launch-count 2 -o gpurun_out/x \\
      python tools/ncu_vcycle.py --config c5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, config_c5, uniform_pm1  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--n", type=int, default=1, help="c5: GPUs the forest is sized for")
ap.add_argument("--passes", type=int, default=-1)
ap.add_argument("--mixed", action="store_true")
ap.add_argument("--eager", action="store_true", help="no CUDA graph")
ap.add_argument("--apply", action="store_true",
                help="profile one plain level operator y = K_L x on the finest level (gmg_level_apply_kernel) "
                     "instead of a V-cycle (the V-cycle runs its residual fused with the restriction)")
args = ap.parse_args()
cfg = config_c5(args.n) if args.config == "c5" else config(args.config)
_, _, h = G.build_config(cfg, passes=args.passes, mixed=args.mixed, graph=not args.eager)
n = h.info()["n_leaf_free"]
b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
for _ in range(3):
    h.vcycle(b, x)
torch.cuda.synchronize()
if args.apply:
    info = h.info()
    L = info["n_levels"] - 1
    xl = torch.rand(info["level_dofs"][L], device="cuda", dtype=torch.float64)
    yl = torch.zeros_like(xl)
    h.level_apply_kernel(L, xl, yl)
    yl.zero_()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    h.level_apply_kernel(L, xl, yl)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
else:
    torch.cuda.profiler.start()
    h.vcycle(b, x)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("levels", h.info()["n_levels"], "gf", h.info()["level_gf"], "r1", h.info()["level_r1"])
