"""Small hot-path runs for compute-sanitizer (tools/sanitize.sh): every kernel
family of the V-cycle on sizes the tools finish in minutes -- 3D Q2 family
patches with edge rows (c3 at 3 passes), grandfamily patches with per-family
coefficients (c4 s=2 lmax=7), the c5 thick-shell recipe, 2D Q2 (c2 truncated),
3D Q1, the mixed-precision cycle, the standalone level operator / transfers and
one CG solve.  No oracle here: parity is the GPU suite's job, this run only has
to touch the kernels' memory and barriers."""
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, uniform_pm1, log_uniform_coef  # noqa: E402

CASES = [("c3", 3, {}, False), ("c4", -1, {"s": 2, "lmax": 6}, False), ("c5", 2, {"shell": (96, 1024)}, False),
         ("c2", -1, {"lmax": 7}, False), ("c3", 3, {"k": 1}, False), ("c3", 3, {}, True), ("c1", -1, {}, False)]
if len(sys.argv) > 1:
    CASES = [CASES[int(a)] for a in sys.argv[1:]]

for name, passes, over, mixed in CASES:
    cfg = dict(config(name))
    cfg.update(over)
    coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"])) if cfg.get("coef") else None
    kw = {} if passes < 0 else {"passes": passes}
    _, _, h = G.build_config(cfg, coef_level2=coef, mixed=mixed, **kw)
    info = h.info()
    n = info["n_leaf_free"]
    b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
    x = torch.zeros_like(b)
    h.vcycle(b, x)                      # eager launches
    h.vcycle(b, x)                      # the captured graph
    L = info["n_levels"] - 1
    for lv in (L, max(1, L - 1)):
        nl = info["level_dofs"][lv]
        xl = torch.tensor(uniform_pm1(nl, stream=3), device="cuda", dtype=torch.float64)
        yl = torch.zeros_like(xl)
        h.level_apply(lv, xl, yl)
    it, rel, _ = h.solve_cg(b, x, rtol=1e-6)
    torch.cuda.synchronize()
    print(f"{name} passes={passes} {over} mixed={mixed}: {n} DoFs, gf={sum(info['level_gf'])}, CG {it} its rel {rel:.2e}",
          flush=True)
    del h
print("sanitize run done")
