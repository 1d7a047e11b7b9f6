"""gmg_vcycle forms the finest level's first pre-smoothing iterate x_1 = c2_0 D^-1 g
(the step from x = 0) inside copy_to_mg (gather_to_mg's x1 arguments)
instead of by a pass over the level that re-reads g.  It is the same expression
on the same values, so the V-cycle must equal the separate pass (GMG_FUSE_X1=0)
up to the order of the operator kernels' L2 reductions (which varies from run to
run: 1e-12 relative in fp64, 2e-6 for the fp32 cycle); the CG's V-cycles (no
copy_to_mg) keep the pass.
Each variant runs in its own process (the switch is read once)."""
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
h.vcycle(b, x)                      # captures the graph
x1 = x.clone()
h.vcycle(b, x)                      # replays it
h.set_eigen(1, 1.7)                 # re-capture with other coefficients
x2 = torch.zeros_like(b)
h.vcycle(b, x2)
xs = torch.zeros_like(b)
it, rel, _ = h.solve_cg(b, xs, rtol=1e-8)
x3 = torch.zeros_like(b)
h.vcycle(b, x3)                     # after the CG captured the plain graph
np.savez({out!r}, x1=x1.cpu().numpy(), x=x.cpu().numpy(), x2=x2.cpu().numpy(), x3=x3.cpu().numpy(),
         xs=xs.cpu().numpy(), it=it, lpv=h.launch_profile()[0])
"""

CASES = [("c3", 3, {}, False), ("c3", 3, {}, True), ("c2", -1, {"lmax": 7}, False), ("c1", -1, {}, False),
         ("c3", 3, {"k": 1}, False)]


def _run(tmp_path, name, passes, over, mixed, on):
    out = str(tmp_path / f"r{on}.npz")
    code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, GMG_FUSE_X1=on), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c3p3", "c3p3-mixed", "c2s", "c1", "c3p3-q1"])
def test_x1_in_copy_to_mg_equals_separate_pass(tmp_path, name, passes, over, mixed):
    on = _run(tmp_path, name, passes, over, mixed, "1")
    off = _run(tmp_path, name, passes, over, mixed, "0")
    assert int(on["lpv"]) == int(off["lpv"]) - 1          # one launch less per V-cycle
    tol = 2e-6 if mixed else 1e-12

    def close(a, b, t=tol):
        return np.abs(a - b).max() <= t * np.abs(b).max()

    for key in ("x1", "x", "x2", "x3"):
        assert close(on[key], off[key]), (key, np.abs(on[key] - off[key]).max() / np.abs(off[key]).max())
    assert close(on["x1"], on["x"]) and close(on["x2"], on["x3"])      # graph replay; after the CG's capture
    assert close(on["xs"], off["xs"], 1e-6)                              # both solved to rtol 1e-8
    assert abs(int(on["it"]) - int(off["it"])) <= 1
