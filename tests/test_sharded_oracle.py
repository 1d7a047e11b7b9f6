"""Sharded execution compared with the ORACLE (VERDICT r1 "sharded
parity against the oracle").

The p-rank V-cycle and GMG-CG, gathered back into the canonical leaf order,
must equal the single-process oracle (oracle/mg.py) to the same bars as the
one-rank path: V-cycle max-norm relative 1e-10, CG iterations +-1 with the true
residual <= 1e-8 (BASELINE.json north_star).  Two transports:

* ranks as host threads of one process (gmg_local_world, stream-ordered
  device copies);
* ranks as separate processes (gmg_host_world, POSIX shared memory,
  host-staged exchanges) -- the same per-rank process flow as the NCCL path,
  runnable on a one-GPU machine.

Eigenvalue estimates are taken from the oracle (gmg_set_eigen on every rank) so
the comparison isolates the sharded V-cycle from the Lanczos estimate, which is
checked separately to 1e-10 (test_gpu_parity.py).  The CPU tests at the end
cover the host-world barrier with two processes (no GPU)."""
import os
import socket
import threading
import uuid

import numpy as np
import pytest

import paper_1904_03317_b200 as G
from gmg_inputs import config, uniform_pm1, log_uniform_coef

VC_TOL = 1e-10


def _cfg(name, k=None):
    if name == "c4s":                       # config-4 recipe, small (variable coefficient)
        cfg = config("c4")
        cfg.update(s=2, lmax=7)
    else:
        cfg = config(name)
    if k is not None:
        cfg["k"] = k
    return cfg


def _coef(cfg):
    if cfg.get("coef") == "level2_log_uniform":
        return log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    return None


_oracle_cache = {}


def _oracle(cfg, coarse="cholesky"):
    from oracle import forest as F, mg
    key = (repr(sorted(cfg.items())), coarse)
    if key not in _oracle_cache:
        of = F.generate(cfg)
        oh = mg.build(of, cfg["k"], coef_level2=_coef(cfg), coarse=coarse)
        b = uniform_pm1(oh.leaf.n_free)
        x_ref = mg.vcycle(oh, b)
        xs_ref, it_ref, _, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
        lams = [oh.levels[l].lam for l in range(1, oh.L + 1)]
        _oracle_cache[key] = (oh, b, x_ref, it_ref, lams)
    return _oracle_cache[key]


def _rel(a, b):
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


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


def _check_against_oracle(n, canon, res, oh, x_ref, it_ref):
    xv = np.full(n, np.nan)
    xsv = np.full(n, np.nan)
    its = set()
    for fo, no, x, xs, it in res:
        xv[canon[fo:fo + no]] = x
        xsv[canon[fo:fo + no]] = xs
        its.add(it)
    assert not np.isnan(xv).any() and not np.isnan(xsv).any()
    assert len(its) == 1, its                       # every rank reports the same count
    it = its.pop()
    assert _rel(xv, x_ref) <= VC_TOL, _rel(xv, x_ref)
    assert abs(it - it_ref) <= 1, (it, it_ref)
    tr = np.linalg.norm(oh.b_leaf - oh.A_leaf @ xsv) / np.linalg.norm(oh.b_leaf)
    assert tr <= 1.01e-8, tr


# ------------------------------------------------------------------ ranks as threads
THREAD_CASES = [("c1", None, 2, "first_child"), ("c1", None, 3, "first_child"), ("c1", None, 4, "first_child"),
                ("c1", None, 8, "first_child"), ("c3p2", None, 2, "first_child"), ("c3p2", None, 4, "first_child"),
                ("c3p2", None, 8, "first_child"), ("c4s", None, 3, "first_child"), ("c4s", None, 8, "first_child"),
                ("c3p2", None, 4, "per_level"), ("c4s", None, 3, "per_level"),
                # 3D Q1 where some ranks have no fused (R1) rows on a level while others do:
                # the prolongation fusion must be decided collectively
                ("brick8", 1, 5, "first_child"), ("c3p2", 1, 32, "first_child")]


# coarse-level gather (gmg_partition_ex): levels with <= coarse cells on rank 0
COARSE_CASES = [("c3p2", None, 4, "first_child", 64), ("c3p2", None, 8, "first_child", 600),
                ("c4s", None, 3, "first_child", 100), ("c1", None, 5, "per_level", 20)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,k,p,mode,coarse", [c + (0,) for c in THREAD_CASES] + COARSE_CASES)
def test_thread_ranks_vs_oracle(name, k, p, mode, coarse):
    import torch
    cfg = _cfg(name, k)
    oh, b_can, x_ref, it_ref, lams = _oracle(cfg)
    world = G.LocalWorld(p)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(lf, p, mode=mode, coarse_cells=coarse)
    if coarse:
        t = part.tallies()
        assert (t[0, 1:] == 0).all() and (t[1, 1:] == 0).all()   # gathered levels on rank 0
    hs = [None] * p
    streams = [torch.cuda.Stream() for _ in range(p)]

    def setup(r):
        def fn():
            torch.cuda.set_device(0)
            hs[r] = G.gmg_setup(lf, part, k=cfg["k"], rank=r, comm=world, coef_level2=_coef(cfg))
            for l, lam in enumerate(lams, start=1):
                hs[r].set_eigen(l, lam)
        return fn

    _run_threads([setup(r) for r in range(p)])
    if name == "brick8" and p == 5:
        r1 = np.array([h.info()["level_r1"] for h in hs])     # [rank, level]
        mixed = [l for l in range(r1.shape[1]) if (r1[:, l] > 0).any() and (r1[:, l] == 0).any()]
        assert mixed, "the case must have a level where only some ranks have R1 rows"
    canon = hs[0].leaf_dofs()[3]
    res = [None] * p

    def work(r):
        def fn():
            torch.cuda.set_device(0)
            fo, no = hs[r].info()["first_owned"], hs[r].n_owned
            s = streams[r]
            with torch.cuda.stream(s):
                b = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
                x = torch.zeros_like(b)
                hs[r].vcycle(b, x, stream=s.cuda_stream)
                rhs = torch.zeros_like(b)
                hs[r].rhs_constant(1.0, rhs, stream=s.cuda_stream)
                xs = torch.zeros_like(b)
                it, _, _ = hs[r].solve_cg(rhs, xs, rtol=1e-8, stream=s.cuda_stream)
                s.synchronize()
            res[r] = (fo, no, x.cpu().numpy(), xs.cpu().numpy(), it)
        return fn

    _run_threads([work(r) for r in range(p)])
    _check_against_oracle(oh.leaf.n_free, canon, res, oh, x_ref, it_ref)
    for h in hs:
        h.close()


# ------------------------------------------------------------------ ranks as processes
def _proc_worker(rank, p, shm, cfg, lams, b_can, q, mode):
    try:
        import torch
        torch.cuda.set_device(0)
        world = G.HostWorld(shm, p, rank, slot_bytes=64 << 20)
        lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
        part = G.gmg_partition(lf, p, mode=mode)
        h = G.gmg_setup(lf, part, k=cfg["k"], rank=rank, comm=world, coef_level2=_coef(cfg), allocator="torch")
        for l, lam in enumerate(lams, start=1):
            h.set_eigen(l, lam)
        canon = h.leaf_dofs()[3]
        fo, no = h.info()["first_owned"], h.n_owned
        b = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
        x = torch.zeros_like(b)
        h.vcycle(b, x)
        rhs = torch.zeros_like(b)
        h.rhs_constant(1.0, rhs)
        xs = torch.zeros_like(b)
        it, _, _ = h.solve_cg(rhs, xs, rtol=1e-8)
        torch.cuda.synchronize()
        out = (fo, no, x.cpu().numpy(), xs.cpu().numpy(), it)
        h.close()
        world.destroy()
        q.put((rank, out, canon if rank == 0 else None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None))


@pytest.mark.gpu
@pytest.mark.parametrize("name,p,mode", [("c1", 2, "first_child"), ("c3p2", 3, "first_child"),
                                         ("c4s", 2, "per_level")])
def test_process_ranks_vs_oracle(name, p, mode):
    import multiprocessing as mp
    cfg = _cfg(name)
    oh, b_can, x_ref, it_ref, lams = _oracle(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shm = "/gmg_test_" + uuid.uuid4().hex[:12]
    ps = [ctx.Process(target=_proc_worker, args=(r, p, shm, cfg, lams, b_can, q, mode)) for r in range(p)]
    for pr in ps:
        pr.start()
    got = [q.get(timeout=600) for _ in ps]
    for pr in ps:
        pr.join(timeout=60)
    errs = [g for g in got if isinstance(g[1], str)]
    assert not errs, errs
    canon = [g[2] for g in got if g[0] == 0][0]
    _check_against_oracle(oh.leaf.n_free, canon, [g[1] for g in got], oh, x_ref, it_ref)


# ------------------------------------------------------------------ CPU: host world plumbing
def _barrier_worker(rank, p, shm, q):
    try:
        w = G.HostWorld(shm, p, rank, slot_bytes=1 << 16)   # collective: returns when all attached
        w.destroy()                                         # collective
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("p", [2, 3])
def test_host_world_attach_and_barrier(p):
    """p processes attach to one shared-memory world and detach collectively (no GPU
    needed: registration with CUDA is optional); the segment is unlinked after."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shm = "/gmg_test_" + uuid.uuid4().hex[:12]
    ps = [ctx.Process(target=_barrier_worker, args=(r, p, shm, q)) for r in range(p)]
    for pr in ps:
        pr.start()
    res = [q.get(timeout=120) for _ in ps]
    for pr in ps:
        pr.join(timeout=30)
    assert all(r[1] == "ok" for r in res), res
    assert not os.path.exists("/dev/shm" + shm)


def test_host_world_rejects_bad_arguments():
    with pytest.raises(G.GmgError):
        G.HostWorld("no_slash", 2, 0)
    with pytest.raises(G.GmgError):
        G.HostWorld("/gmg_x", 2, 5)


# ------------------------------------------------------------------ rank-local builds vs the oracle
RL_CASES = [("c1", None, 3, "first_child", 0), ("c3p2", None, 4, "first_child", 0),
            ("c3p2", None, 8, "first_child", 0), ("c4s", None, 3, "per_level", 0), ("brick8", 1, 5, "first_child", 0),
            ("c3p2", None, 8, "first_child", 600)]


@pytest.mark.gpu
@pytest.mark.parametrize("name,k,p,mode,coarse", RL_CASES)
def test_rank_local_threads_vs_oracle(name, k, p, mode, coarse):
    """GMG_RANK_LOCAL hierarchies (no global numbering; inputs and outputs
    matched by node key) against the oracle: V-cycle 1e-10, CG +-1 / 1e-8."""
    import torch
    from gmg_inputs import uniform_pm1_keys
    cfg = _cfg(name, k)
    oh, _, _, it_ref, lams = _oracle(cfg)
    from oracle import mg
    okeys = oh.leaf.key[oh.leaf.free_index >= 0].astype(np.uint64)        # canonical (Morton) order
    b_ref = uniform_pm1_keys(okeys)
    x_ref = mg.vcycle(oh, b_ref)
    world = G.LocalWorld(p)
    lf = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(lf, p, mode=mode, coarse_cells=coarse)
    hs = [None] * p
    streams = [torch.cuda.Stream() for _ in range(p)]

    def setup(r):
        def fn():
            torch.cuda.set_device(0)
            hs[r] = G.gmg_setup(lf, part, k=cfg["k"], rank=r, comm=world, coef_level2=_coef(cfg), rank_local=True)
            for l, lam in enumerate(lams, start=1):
                hs[r].set_eigen(l, lam)
        return fn

    _run_threads([setup(r) for r in range(p)])
    assert hs[0].info()["n_leaf_free"] == oh.leaf.n_free
    res = [None] * p

    def work(r):
        def fn():
            torch.cuda.set_device(0)
            keys, _ = hs[r].owned_leaf_keys()
            s = streams[r]
            with torch.cuda.stream(s):
                b = torch.tensor(uniform_pm1_keys(keys), device="cuda", dtype=torch.float64)
                x = torch.zeros_like(b)
                hs[r].vcycle(b, x, stream=s.cuda_stream)
                rhs = torch.zeros_like(b)
                hs[r].rhs_constant(1.0, rhs, stream=s.cuda_stream)
                xs = torch.zeros_like(b)
                it, _, _ = hs[r].solve_cg(rhs, xs, rtol=1e-8, stream=s.cuda_stream)
                s.synchronize()
            res[r] = (keys, x.cpu().numpy(), xs.cpu().numpy(), it)
        return fn

    _run_threads([work(r) for r in range(p)])
    keys = np.concatenate([q[0] for q in res])
    order = np.argsort(keys)
    assert np.array_equal(keys[order], okeys)
    xv = np.concatenate([q[1] for q in res])[order]
    xsv = np.concatenate([q[2] for q in res])[order]
    assert len({q[3] for q in res}) == 1
    assert _rel(xv, x_ref) <= VC_TOL, _rel(xv, x_ref)
    assert abs(res[0][3] - it_ref) <= 1
    tr = np.linalg.norm(oh.b_leaf - oh.A_leaf @ xsv) / np.linalg.norm(oh.b_leaf)
    assert tr <= 1.01e-8, tr
    for h in hs:
        h.close()
