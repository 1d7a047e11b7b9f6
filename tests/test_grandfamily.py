"""Grandfamily patches (kernels.cuh gfam_tensor_apply, plan.hpp): where the 8
families below one level-(l-2) cell are all local and share one coefficient,
the level operator runs as one Kronecker sum on their (4k+1)^3 patch.  This is
the same operator (the sum of the 64 cell operators), so results must agree with
the family-patch path (GMG_GFAM=0) up to summation order -- 1e-13 relative for
fp64, 2e-6 for the fp32 V-cycle -- and the V-cycle with grandfamilies must match
the oracle at the north_star bar (1e-10).  Each variant runs in its own process
(GMG_GFAM is read at gmg_setup)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1904_03317_b200 as G
from gmg_inputs import config, uniform_pm1, log_uniform_coef
cfg = dict(config({name!r})); cfg.update({over!r})
coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"])) if cfg.get("coef") else None
_, _, h = G.build_config(cfg, passes={passes}, coef_level2=coef, mixed={mixed})
info = h.info()
n = info["n_leaf_free"]
b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
h.vcycle(b, x)
L = info["n_levels"] - 1
nl = info["level_dofs"][L]
xl = torch.tensor(uniform_pm1(nl, stream=3), device="cuda", dtype=torch.float64)
yl = torch.zeros_like(xl)
h.level_apply(L, xl, yl)
rhs = torch.zeros_like(b)
h.rhs_constant(1.0, rhs)
xs = torch.zeros_like(b)
it, rel, _ = h.solve_cg(rhs, xs, rtol=1e-8)
np.savez({out!r}, x=x.cpu().numpy(), y=yl.cpu().numpy(), xs=xs.cpu().numpy(), it=it,
         gf=np.array(info["level_gf"]), r1=np.array(info["level_r1"]), fam=np.array(info["level_families"]))
"""

CASES = [("c4", -1, {"s": 2, "lmax": 7}, False), ("c4", -1, {"s": 2, "lmax": 7}, True),
         ("c5", 2, {"shell": (96, 1024)}, False), ("c3", 4, {}, False)]


def _run(tmp_path, name, passes, over, mixed, gfam):
    out = str(tmp_path / f"r{gfam}.npz")
    code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
    env = dict(os.environ, GMG_GFAM=gfam)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c4s", "c4s-mixed", "c5-thick-p2", "c3p4"])
def test_grandfamily_matches_family_path(tmp_path, name, passes, over, mixed):
    on = _run(tmp_path, name, passes, over, mixed, "1")
    off = _run(tmp_path, name, passes, over, mixed, "0")
    assert off["gf"].sum() == 0
    if name != "c3":
        assert on["gf"].sum() > 0, "the case must contain complete grandfamilies"
        assert on["r1"].sum() > off["r1"].sum()     # grandfamily interiors are complete rows
    tol = 2e-6 if mixed else 1e-13
    for key in ("x", "y"):
        a, b = on[key], off[key]
        assert np.abs(a - b).max() <= tol * np.abs(b).max(), (key, np.abs(a - b).max() / np.abs(b).max())
    assert abs(int(on["it"]) - int(off["it"])) <= (1 if mixed else 0)
    assert np.abs(on["xs"] - off["xs"]).max() <= 1e-9 * np.abs(off["xs"]).max()


def test_grandfamily_vcycle_vs_oracle():
    """c4s V-cycle with grandfamily patches against the oracle (eigenvalues from
    the oracle), 1e-10."""
    import torch
    import paper_1904_03317_b200 as G
    from gmg_inputs import config, uniform_pm1, log_uniform_coef
    from oracle import forest as F, mg
    cfg = dict(config("c4"))
    cfg.update(s=2, lmax=7)
    coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    _, _, h = G.build_config(cfg, coef_level2=coef)
    assert sum(h.info()["level_gf"]) > 0
    oh = mg.build(F.generate(cfg), cfg["k"], coef_level2=coef)
    for l in range(1, oh.L + 1):
        h.set_eigen(l, oh.levels[l].lam)
    b = uniform_pm1(oh.leaf.n_free)
    x = torch.zeros(oh.leaf.n_free, device="cuda", dtype=torch.float64)
    h.vcycle(torch.tensor(b, device="cuda", dtype=torch.float64), x)
    ref = mg.vcycle(oh, b)
    err = np.abs(x.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 1e-10, err


@pytest.mark.parametrize("name,passes,over", [("c3", 3, {}), ("c5", 2, {"shell": (96, 1024)})], ids=["c3p3", "c5-thick"])
def test_z1_step_matches_separate_pass(tmp_path, name, passes, over):
    """TA_CHEB_Z1 (x_1 formed inside the step-1 kernels, GMG_Z1=1) gives the
    V-cycle of the separate pass + TA_CHEB_X1."""
    outs = []
    for z1 in ("1", "0"):
        out = str(tmp_path / f"z{z1}.npz")
        code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=False, out=out)
        env = dict(os.environ, GMG_Z1=z1)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(np.load(out))
    a, b = outs[0]["x"], outs[1]["x"]
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
    assert int(outs[0]["it"]) == int(outs[1]["it"])
