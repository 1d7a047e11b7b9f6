"""The V-cycle's residual and restriction fused into one operator pass
(kernels.cuh TA_RES, device.cu res_restrict): d_{l-1} += P^T (d_l - K_l x_l)
with each family / grandfamily patch restricting its own operator contribution
and d on the nodes it transfer-owns (R26).  By linearity
this is the separate path's P^T (d - t) with t = K x summed first
(GMG_FUSE_RES=0: plain operator, export-add of t, warp_restrict), up to the
order of the additions.  Runs the V-cycle in two processes and compares at
1e-13 relative (fp64; 2e-6 for the fp32 V-cycle), the same bar as the fused
prolongation: a dropped term, a wrong weight or a double-counted d shows up
orders of magnitude above it.  Cases cover family patches (c3p4, Q1 and Q2),
per-family coefficients (c4s) and grandfamily patches (c5 recipe, thick shell)."""
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
from gmg_inputs import config, uniform_pm1, log_uniform_coef
cfg = dict(config({name!r})); cfg.update({over!r})
coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"])) if cfg.get("coef") else None
_, _, h = G.build_config(cfg, passes={passes}, coef_level2=coef, mixed={mixed})
n = h.info()["n_leaf_free"]
b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
h.vcycle(b, x)
h.vcycle(b, x)
kinds = sorted({{r["kind"] for r in h.profile_vcycle(b, torch.zeros_like(b), n_rep=1) if r["launches"]}})
np.save({out!r}, x.cpu().numpy())
print("KINDS", ",".join(kinds))
"""

CASES = [("c3", 4, {}, False), ("c3", 4, {}, True), ("c4", -1, {"s": 2, "lmax": 7}, False),
         ("c3", 4, {"k": 1}, False), ("c5", 2, {"shell": (96, 1024)}, False), ("c2", -1, {}, False),
         ("c1", -1, {}, False)]


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c3p4", "c3p4-mixed", "c4s", "c3p4-k1", "c5-thick-p2", "c2-2d-q2", "c1-2d-q1"])
def test_fused_residual_matches_separate(tmp_path, name, passes, over, mixed):
    outs, kinds = [], []
    for fuse in ("1", "0"):
        out = str(tmp_path / f"x{fuse}.npy")
        code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
        env = dict(os.environ, GMG_FUSE_RES=fuse)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
        kinds.append([ln for ln in r.stdout.splitlines() if ln.startswith("KINDS")][0].split()[1].split(","))
    # the fused kind runs in the first cycle only (levels without tensor kernels keep the separate path)
    assert "res_restrict" in kinds[0], kinds[0]
    assert "res_restrict" not in kinds[1] and "restrict" in kinds[1], kinds[1]
    err = np.abs(outs[0] - outs[1]).max() / np.abs(outs[1]).max()
    assert err < (2e-6 if mixed else 1e-13), err
    assert np.abs(outs[0]).max() > 0
