"""The persistent small-level kernel (kernels.cuh small_vcycle, opt-in with
GMG_SLK=1): V(l_s) in one cooperative kernel gives the V-cycle of the per-step
kernels (same device bodies, same order; the reductions of shared rows add in
L2 order, so 1e-13 relative), for 2D and 3D, Q1 and Q2, fp64 and fp32."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1904_03317_b200 as G
from gmg_inputs import config, uniform_pm1
cfg = dict(config({name!r})); cfg.update({over!r})
_, _, h = G.build_config(cfg, passes={passes}, mixed={mixed})
n = h.info()["n_leaf_free"]
b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
h.vcycle(b, x)
h.vcycle(b, x)
xe = torch.zeros_like(b)
rhs = torch.zeros_like(b)
h.rhs_constant(1.0, rhs)
it, _, _ = h.solve_cg(rhs, xe, rtol=1e-8)
np.savez({out!r}, x=x.cpu().numpy(), it=it, sl=h.info()["small_levels"])
"""

CASES = [("c1", -1, {}, False), ("c3", 3, {}, False), ("c3", 3, {}, True), ("c3", 3, {"k": 1}, False),
         ("c2", -1, {"lmax": 9}, False)]


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c1", "c3p3", "c3p3-mixed", "c3p3-k1", "c2-small"])
def test_small_level_kernel_matches_per_step_kernels(tmp_path, name, passes, over, mixed):
    outs = []
    for slk in ("1", "0"):
        out = str(tmp_path / f"x{slk}.npz")
        code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
        env = dict(os.environ, GMG_SLK=slk)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    assert int(outs[0]["sl"]) > 0 and int(outs[1]["sl"]) == 0
    a, b = outs[0]["x"], outs[1]["x"]
    assert np.abs(a - b).max() <= (2e-6 if mixed else 1e-13) * np.abs(b).max()
    assert abs(int(outs[0]["it"]) - int(outs[1]["it"])) <= (1 if mixed else 0)
