import os, sys, subprocess, numpy as np
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1904_03317_b200 as G
from gmg_inputs import config, uniform_pm1
cfg = dict(config("c3"))
_, _, h = G.build_config(cfg, passes=4)
n = h.info()["n_leaf_free"]
b = torch.tensor(uniform_pm1(n), device="cuda", dtype=torch.float64)
x = torch.zeros_like(b)
h.vcycle(b, x)
np.save(sys.argv[1], x.cpu().numpy())
L = h.info()["n_levels"] - 1
'''
outs = []
for f in (sys.argv[1], sys.argv[2]):
    out = f"/tmp/diag_{f}_{len(outs)}.npy"
    r = subprocess.run([sys.executable, "-c", code, out], env=dict(os.environ, GMG_FUSE_PROLONG=f), capture_output=True, text=True)
    print(r.returncode, r.stderr[-500:])
    outs.append(np.load(out))
d = np.abs(outs[0] - outs[1])
print("max abs diff", d.max(), "rel", d.max() / np.abs(outs[1]).max(), "n differing", (d > 0).sum(), "of", len(d))
