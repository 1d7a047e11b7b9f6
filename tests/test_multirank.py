"""Multi-rank path: rank-local layouts and ghost sets (CPU,
bit-exact vs an oracle computation), a world_size-2 gloo run of the host logic
(CPU), and the full V-cycle / CG with p logical ranks as host threads on one
GPU (ThreadComm transport) compared with the single-rank result."""
import os
import socket
import threading

import numpy as np
import pytest

import paper_1904_03317_b200 as G
from oracle import forest as F, mg
from oracle.spaces import parent_owner
from gmg_inputs import config, uniform_pm1, log_uniform_coef


# ------------------------------------------------------------------ oracle ghost sets
def oracle_rank_layout(f, k, p):
    """Per level and rank: owned global range and ghost global indices, from the
    definitions (R25/R26): rank q computes the families whose parent it
    owns (level 0: the cells it owns); it needs their nodes and the nodes of the
    parents of its next-finer families; ghosts = needed DoFs owned by others."""
    T = mg.topology(f, k, p)
    cells = T.cells
    out = []
    for l, s in enumerate(T.spaces):
        go = s.global_order()                       # global position -> canonical
        glob_of = np.empty(max(s.n, 1), dtype=np.int64)
        glob_of[go] = np.arange(s.n)
        own_glob = s.owner[go]
        if l == 0:
            comp = cells[0].owner
        else:
            comp = parent_owner(cells[l], cells[l - 1])
        needed = [set() for _ in range(p)]
        cd = s.cell_dofs
        for c in range(cd.shape[0]):
            for i in cd[c]:
                if i >= 0:
                    needed[comp[c]].add(int(glob_of[i]))
        if l + 1 < len(T.spaces):
            # parents of next-finer cells: computed by the owner of the parent
            fine = cells[l + 1]
            R = int(max(fine.gc.max(initial=0), cells[l].gc.max(initial=0))) + 3
            key = lambda g: sum(((g[:, j] + 1) * R ** j) for j in range(g.shape[1]))
            pk = key(cells[l].gc)
            o = np.argsort(pk)
            par = o[np.searchsorted(pk[o], key(fine.gc >> 1))]
            for c in np.unique(par):
                q = cells[l].owner[c]
                for i in cd[c]:
                    if i >= 0:
                        needed[q].add(int(glob_of[i]))
        lv = []
        for q in range(p):
            owned = np.nonzero(own_glob == q)[0]
            first = int(owned[0]) if owned.size else int(np.searchsorted(own_glob, q))
            gh = sorted(g for g in needed[q] if own_glob[g] != q)
            lv.append((first, int(owned.size), np.array(gh, dtype=np.int64)))
        out.append(lv)
    return out


@pytest.mark.parametrize("name,k,p", [("c1", 1, 2), ("c1", 1, 5), ("c3p2", 2, 3), ("c1", 2, 8)])
def test_rank_layout_matches_oracle(name, k, p):
    cfg = dict(config(name))
    f = F.generate(cfg)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(lf, p)
    ref = oracle_rank_layout(f, k, p)
    for r in range(p):
        h = G.gmg_setup(lf, part, k=k, rank=r, host_only=True)
        for l in range(len(ref)):
            fo, no, gh = h.rank_level(l)
            assert (fo, no) == ref[l][r][:2] or (no == 0 and ref[l][r][1] == 0), (l, r)
            assert np.array_equal(gh, ref[l][r][2]), (l, r)


# ------------------------------------------------------------------ gloo, world size 2
def _gloo_worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = config(name)
        lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
        part = G.gmg_partition(lf, world)
        h = G.gmg_setup(lf, part, k=cfg["k"], rank=rank, host_only=True)
        info = h.info()
        mine = {"leaf": (info["first_owned"], info["n_owned"]), "levels": []}
        for l in range(info["n_levels"]):
            fo, no, gh = h.rank_level(l)
            mine["levels"].append((fo, no, gh.tolist()))
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        n_leaf = info["n_leaf_free"]
        # leaf ownership ranges tile the global leaf numbering
        rng = sorted(a["leaf"] for a in allv)
        pos = 0
        for fo, no in rng:
            assert fo == pos or no == 0
            pos += no
        assert pos == n_leaf
        for l in range(info["n_levels"]):
            total = info["level_dofs"][l]
            owned = sorted((a["levels"][l][0], a["levels"][l][1]) for a in allv)
            pos = 0
            for fo, no in owned:
                assert fo == pos or no == 0
                pos += no
            assert pos == total
            # every ghost of rank r is owned by the other rank
            for r, a in enumerate(allv):
                for g in a["levels"][l][2]:
                    other = allv[1 - r]["levels"][l]
                    assert other[0] <= g < other[0] + other[1]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("name", ["c1", "c3p2"])
def test_gloo_world_size_2_layout(name):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    res = [q.get(timeout=300) for _ in ps]
    for p_ in ps:
        p_.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


# ------------------------------------------------------------------ GPU: ranks as threads
def _run_threads(fns):
    errs = []

    def wrap(fn):
        try:
            fn()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(fn,)) for fn in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def _coef(cfg):
    if cfg.get("coef") == "level2_log_uniform":       # config 4: a per level-2 cell, SFC order
        return log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    return None


def _local_group(cfg, p, **kw):
    import torch
    world = G.LocalWorld(p)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(lf, p)
    hs = [None] * p
    streams = [torch.cuda.Stream() for _ in range(p)]

    def setup(r):
        def fn():
            torch.cuda.set_device(0)
            hs[r] = G.gmg_setup(lf, part, k=cfg["k"], rank=r, comm=world, coef_level2=_coef(cfg), **kw)
        return fn

    _run_threads([setup(r) for r in range(p)])
    return world, lf, part, hs, streams


@pytest.mark.gpu
def test_nccl_transport_loads():
    """libnccl is dlopen'ed (the torch copy) and a 1-rank communicator initialises."""
    uid = G.gmg_nccl_get_unique_id()
    assert len(uid) == 128
    c = G.NcclComm(uid, 1, 0)
    assert c.h
    c.destroy()


@pytest.mark.gpu
@pytest.mark.parametrize("name,p", [("c1", 2), ("c1", 3), ("c3p2", 2), ("c3p2", 4), ("c2", 3), ("c4s", 3),
                                    ("brick8-cheb", 3), ("brick8-cheb", 5)])
def test_local_ranks_equal_single_rank(name, p):
    import torch
    kw = {}
    if name == "c4s":      # config-4 recipe at a small size (variable coefficient)
        cfg = config("c4")
        cfg.update(s=2, lmax=7)
    elif name == "brick8-cheb":   # multi-cell coarse mesh, collective Chebyshev coarse solver
        cfg = config("brick8")
        kw = {"coarse": "chebyshev"}
    else:
        cfg = config(name)
    _, _, h1 = G.build_config(cfg, coef_level2=_coef(cfg), **kw)
    n = h1.info()["n_leaf_free"]
    canon1 = h1.leaf_dofs()[3]
    b_can = uniform_pm1(n)
    b1 = torch.tensor(b_can[canon1], device="cuda", dtype=torch.float64)
    x1 = torch.zeros_like(b1)
    h1.vcycle(b1, x1)
    rhs1 = torch.zeros_like(b1)
    h1.rhs_constant(1.0, rhs1)
    xs1 = torch.zeros_like(b1)
    it1, _, _ = h1.solve_cg(rhs1, xs1, rtol=1e-8)
    ref_x = np.empty(n)
    ref_x[canon1] = x1.cpu().numpy()
    ref_s = np.empty(n)
    ref_s[canon1] = xs1.cpu().numpy()

    world, lf, part, hs, streams = _local_group(cfg, p, **kw)
    canon = hs[0].leaf_dofs()[3]
    res = [None] * p

    def work(r):
        def fn():
            torch.cuda.set_device(0)
            info = hs[r].info()
            fo, no = info["first_owned"], info["n_owned"]
            with torch.cuda.stream(streams[r]):
                b = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
                x = torch.zeros_like(b)
                hs[r].vcycle(b, x, stream=streams[r].cuda_stream)
                rhs = torch.zeros_like(b)
                hs[r].rhs_constant(1.0, rhs, stream=streams[r].cuda_stream)
                xs = torch.zeros_like(b)
                it, rel, _ = hs[r].solve_cg(rhs, xs, rtol=1e-8, stream=streams[r].cuda_stream)
                streams[r].synchronize()
            res[r] = (fo, no, x.cpu().numpy(), xs.cpu().numpy(), it)
        return fn

    _run_threads([work(r) for r in range(p)])
    xv = np.empty(n)
    xsv = np.empty(n)
    for fo, no, x, xs, it in res:
        xv[canon[fo:fo + no]] = x
        xsv[canon[fo:fo + no]] = xs
        assert it == it1
    assert np.abs(xv - ref_x).max() <= 1e-12 * np.abs(ref_x).max()
    assert np.abs(xsv - ref_s).max() <= 1e-9 * np.abs(ref_s).max()


@pytest.mark.gpu
@pytest.mark.parametrize("name,p", [("c3p2", 3), ("c4s", 2)])
def test_local_ranks_mixed_precision(name, p):
    """The fp32 V-cycle (R13) sharded over p local ranks (fp64 wire format for the
    ghost values) equals the single-rank fp32 V-cycle up to fp32 rounding (the
    reductions of shared rows add in a different order), and its CG converges in
    the same number of iterations."""
    import torch
    if name == "c4s":
        cfg = config("c4")
        cfg.update(s=2, lmax=7)
    else:
        cfg = config(name)
    _, _, h1 = G.build_config(cfg, coef_level2=_coef(cfg), mixed=True)
    n = h1.info()["n_leaf_free"]
    canon1 = h1.leaf_dofs()[3]
    b_can = uniform_pm1(n)
    b1 = torch.tensor(b_can[canon1], device="cuda", dtype=torch.float64)
    x1 = torch.zeros_like(b1)
    h1.vcycle(b1, x1)
    rhs1 = torch.zeros_like(b1)
    h1.rhs_constant(1.0, rhs1)
    it1, _, _ = h1.solve_cg(rhs1, torch.zeros_like(b1), rtol=1e-8)
    ref_x = np.empty(n)
    ref_x[canon1] = x1.cpu().numpy()

    world, lf, part, hs, streams = _local_group(cfg, p, mixed=True)
    canon = hs[0].leaf_dofs()[3]
    res = [None] * p

    def work(r):
        def fn():
            torch.cuda.set_device(0)
            info = hs[r].info()
            fo, no = info["first_owned"], info["n_owned"]
            with torch.cuda.stream(streams[r]):
                b = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
                x = torch.zeros_like(b)
                hs[r].vcycle(b, x, stream=streams[r].cuda_stream)
                rhs = torch.zeros_like(b)
                hs[r].rhs_constant(1.0, rhs, stream=streams[r].cuda_stream)
                it, _, _ = hs[r].solve_cg(rhs, torch.zeros_like(b), rtol=1e-8, stream=streams[r].cuda_stream)
                streams[r].synchronize()
            res[r] = (fo, no, x.cpu().numpy(), it)
        return fn

    _run_threads([work(r) for r in range(p)])
    xv = np.empty(n)
    for fo, no, x, it in res:
        xv[canon[fo:fo + no]] = x
        assert abs(it - it1) <= 1
    assert np.abs(xv - ref_x).max() <= 2e-5 * np.abs(ref_x).max()
