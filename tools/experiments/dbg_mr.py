import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1904_03317_b200 as G
from gmg_inputs import config, uniform_pm1
from test_multirank import _local_group, _run_threads
name = sys.argv[1]; p = int(sys.argv[2])
cfg = config(name)
_, _, h1 = G.build_config(cfg)
L = h1.info()["n_levels"]
lam1 = [h1.get_eigen(l) for l in range(1, L)]
n = h1.info()["n_leaf_free"]; canon1 = h1.leaf_dofs()[3]; b_can = uniform_pm1(n)
b1 = torch.tensor(b_can[canon1], device="cuda", dtype=torch.float64); x1 = torch.zeros_like(b1)
h1.vcycle(b1, x1); ref = np.empty(n); ref[canon1] = x1.cpu().numpy()
for trial in range(3):
    world, lf, part, hs, streams = _local_group(cfg, p)
    lamp = [[hs[r].get_eigen(l) for l in range(1, L)] for r in range(p)]
    print("eig rel diff per level (rank0):", np.max(np.abs(np.array(lamp[0]) - lam1) / np.abs(lam1)))
    canon = hs[0].leaf_dofs()[3]
    for force in (False, True):
        if force:
            for r in range(p):
                for l in range(1, L): hs[r].set_eigen(l, lam1[l - 1])
        res = [None] * p
        def work(r):
            def fn():
                torch.cuda.set_device(0)
                info = hs[r].info(); fo, no = info["first_owned"], info["n_owned"]
                with torch.cuda.stream(streams[r]):
                    b = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
                    x = torch.zeros_like(b)
                    hs[r].vcycle(b, x, stream=streams[r].cuda_stream)
                    streams[r].synchronize()
                res[r] = (fo, no, x.cpu().numpy())
            return fn
        _run_threads([work(r) for r in range(p)])
        xv = np.empty(n)
        for fo, no, x in res: xv[canon[fo:fo + no]] = x
        print(f"trial {trial} force_eig={force}: vcycle rel err {np.abs(xv - ref).max() / np.abs(ref).max():.3e}")
