"""The prolongation fused into the first post-smoothing step (kernels.cuh,
TA_CHEB_P01) gives the V-cycle of the separate prolongation kernel: a fine node
shared by families of different parents gets P x_{l-1} from either parent with
the same arithmetic (exact picks across the shared coordinate).  Runs the
V-cycle in two processes (GMG_FUSE_PROLONG=1 / 0) and compares.  The V-cycle is
not bitwise reproducible run to run (rows reduced by several family patches
add in the order the REDs reach L2; measured 7e-16 relative on c3p4), so the
bar is 1e-13 relative in the max norm (fp64; 2e-6 = ~30 ulp for the fp32
V-cycle) — a wrong fused term shows up orders of magnitude above it."""
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
np.save({out!r}, x.cpu().numpy())
"""

CASES = [("c3", 4, {}, False), ("c3", 4, {}, True), ("c4", -1, {"s": 2, "lmax": 7}, False), ("c3", 4, {"k": 1}, False)]


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c3p4", "c3p4-mixed", "c4s", "c3p4-k1"])
def test_fused_prolongation_matches_separate(tmp_path, name, passes, over, mixed):
    outs = []
    for fuse in ("1", "0"):
        out = str(tmp_path / f"x{fuse}.npy")
        code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
        env = dict(os.environ, GMG_FUSE_PROLONG=fuse)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    err = np.abs(outs[0] - outs[1]).max() / np.abs(outs[1]).max()
    assert err < (2e-6 if mixed else 1e-13), err
    assert np.abs(outs[0]).max() > 0
