"""Float parity of the CUDA path (through the C ABI) against the oracle.

Bars (BASELINE.json north_star): operator applies / transfers / diagonal /
leaf operator 1e-12 relative (max-norm, reading R23), one V-cycle 1e-10,
CG iterations +-1 at 1e-8.  Inputs: uniform[-1,1) by canonical index
(gmg_inputs, seed 190403317).  With p = 1 the library's global level/leaf
order equals the canonical (Morton) order of the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, uniform_pm1, log_uniform_coef, STREAM_PROBE  # noqa: E402
from oracle import forest as F, mg  # noqa: E402

OP_TOL = 1e-12
VC_TOL = 1e-10


def dev(a):
    return torch.tensor(np.asarray(a), device="cuda", dtype=torch.float64)


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


_cache = {}


def pair(name, k=None, passes=-1, cfg_over=None):
    key = (name, k, passes, tuple(sorted((cfg_over or {}).items())))
    if key in _cache:
        return _cache[key]
    cfg = dict(config(name))
    if cfg_over:
        cfg.update(cfg_over)
    if k is not None:
        cfg["k"] = k
    coef = None
    if cfg.get("coef") == "level2_log_uniform":       # config 4: a per level-2 cell, SFC order
        coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
    f, part, h = G.build_config(cfg, passes=passes, coef_level2=coef)
    of = F.generate(cfg, passes=passes)
    oh = mg.build(of, cfg["k"], coef_level2=coef)
    _cache[key] = (h, oh, (f, part))
    return _cache[key]


# c4s: the config-4 recipe (variable coefficient, corner-graded) at a small size
# (s = 2, lmax = 7): levels 0-1 exact sub-box matrices, level 2 per-cell and
# levels >= 3 per-family coefficients are all exercised.
C4S = {"s": 2, "lmax": 7}
CASES = [("c1", None), ("c1", 2), ("c3p2", None), ("c3p2", 1), ("c4", None, -1, C4S), ("c4", 1, -1, C4S)]


@pytest.fixture(scope="module", params=CASES,
                ids=[f"{c[0]}{'s' if len(c) > 2 else ''}-k{c[1]}" for c in CASES])
def hp(request):
    return pair(*request.param)


def test_sizes_match(hp):
    h, oh, _ = hp
    info = h.info()
    assert info["n_levels"] == oh.L + 1
    assert info["n_leaf_free"] == oh.leaf.n_free
    for l, lev in enumerate(oh.levels):
        assert info["level_dofs"][l] == lev.space.n


def test_level_apply(hp):
    h, oh, _ = hp
    off = 0
    for l, lev in enumerate(oh.levels):
        n = lev.space.n
        if n == 0:
            continue
        x = uniform_pm1(n, STREAM_PROBE, offset=off)
        off += n
        y = torch.zeros(n, device="cuda", dtype=torch.float64)
        h.level_apply(l, dev(x), y)
        assert rel(y.cpu().numpy(), lev.K @ x) < OP_TOL, l


def test_diagonal(hp):
    h, oh, _ = hp
    for l, lev in enumerate(oh.levels):
        n = lev.space.n
        if n == 0:
            continue
        d = torch.zeros(n, device="cuda", dtype=torch.float64)
        h.level_diagonal(l, d)
        ref = np.where(lev.S, lev.K.diagonal(), 0.0)
        assert rel(d.cpu().numpy(), ref) < OP_TOL


def test_transfers_and_adjointness(hp):
    h, oh, _ = hp
    for l in range(1, oh.L + 1):
        P = oh.levels[l].P
        nf, nc = P.shape
        if nf == 0 or nc == 0:
            continue
        xc = uniform_pm1(nc, STREAM_PROBE, offset=7 * l)
        rf = uniform_pm1(nf, STREAM_PROBE, offset=1000 + 7 * l)
        xf = torch.zeros(nf, device="cuda", dtype=torch.float64)
        h.prolongate(l, dev(xc), xf)
        assert rel(xf.cpu().numpy(), P @ xc) < OP_TOL
        dc = torch.zeros(nc, device="cuda", dtype=torch.float64)
        h.restrict(l, dev(rf), dc)
        assert rel(dc.cpu().numpy(), P.T @ rf) < OP_TOL
        # <R r, x> = <r, P x> (R = P^T)
        lhs = float(dc.cpu().numpy() @ xc)
        rhs = float(rf @ xf.cpu().numpy())
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_leaf_apply_and_rhs(hp):
    h, oh, _ = hp
    n = oh.leaf.n_free
    u = uniform_pm1(n, STREAM_PROBE, offset=99)
    v = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.leaf_apply(dev(u), v)
    assert rel(v.cpu().numpy(), oh.A_leaf @ u) < OP_TOL
    b = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, b)
    assert rel(b.cpu().numpy(), oh.b_leaf) < OP_TOL


def test_eigen_estimates(hp):
    h, oh, _ = hp
    for l in range(1, oh.L + 1):
        ref = oh.levels[l].lam
        got = h.get_eigen(l)
        assert abs(got - ref) <= 1e-10 * max(ref, 1e-300), (l, got, ref)


def test_smoother(hp):
    h, oh, _ = hp
    for l in range(1, oh.L + 1):
        lev = oh.levels[l]
        n = lev.space.n
        if not lev.S.any():
            continue
        h.set_eigen(l, lev.lam)
        g = uniform_pm1(n, STREAM_PROBE, offset=3 * l) * (lev.S | lev.E)
        x0 = uniform_pm1(n, STREAM_PROBE, offset=5000 + 3 * l)
        x = dev(x0)
        h.level_smooth(l, dev(g), x, False)
        ref = mg.chebyshev(lev, g, x0, oh.degree)
        assert rel(x.cpu().numpy(), ref) < VC_TOL
        x = torch.zeros(n, device="cuda", dtype=torch.float64)
        h.level_smooth(l, dev(g), x, True)
        ref = mg.chebyshev(lev, g, None, oh.degree)
        assert rel(x.cpu().numpy(), ref) < VC_TOL


def test_vcycle(hp):
    h, oh, _ = hp
    for l in range(1, oh.L + 1):
        h.set_eigen(l, oh.levels[l].lam)
    n = oh.leaf.n_free
    b = uniform_pm1(n)
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.vcycle(dev(b), x)
    assert rel(x.cpu().numpy(), mg.vcycle(oh, b)) < VC_TOL
    # zero in, zero out; linearity
    z = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.vcycle(torch.zeros(n, device="cuda", dtype=torch.float64), z)
    assert float(z.abs().max()) == 0.0
    x2 = torch.zeros_like(x)
    h.vcycle(dev(2.5 * b), x2)
    assert rel(x2.cpu().numpy(), 2.5 * x.cpu().numpy()) < 1e-13


def test_cg_iterations(hp):
    h, oh, _ = hp
    n = oh.leaf.n_free
    b = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, b)
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    it, relres, _ = h.solve_cg(b, x, rtol=1e-8)
    xo, it_ref, rel_ref, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
    assert abs(it - it_ref) <= 1, (it, it_ref)
    assert relres <= 1e-8
    tr = np.linalg.norm(oh.b_leaf - oh.A_leaf @ x.cpu().numpy()) / np.linalg.norm(oh.b_leaf)
    assert tr <= 1.01e-8
    assert rel(x.cpu().numpy(), xo) < 1e-6


def test_cg_not_converged_and_zero_rhs():
    h, oh, _ = pair("c1")
    n = oh.leaf.n_free
    b = dev(uniform_pm1(n))
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    it, relres, code = h.solve_cg(b, x, rtol=1e-30, max_it=3, raise_on_fail=False)
    assert code == 9 and it == 3 and relres > 0
    it, relres, code = h.solve_cg(torch.zeros(n, device="cuda", dtype=torch.float64), x, rtol=1e-8)
    assert it == 0 and float(x.abs().max()) == 0.0


def test_graph_and_eager_agree():
    cfg = config("c1")
    _, _, h1 = G.build_config(cfg, graph=True)
    _, _, h2 = G.build_config(cfg, graph=False)
    n = h1.info()["n_leaf_free"]
    b = dev(uniform_pm1(n))
    x1 = torch.zeros(n, device="cuda", dtype=torch.float64)
    x2 = torch.zeros(n, device="cuda", dtype=torch.float64)
    h1.vcycle(b, x1)
    h1.vcycle(b, x1)
    h2.vcycle(b, x2)
    assert rel(x1.cpu().numpy(), x2.cpu().numpy()) < 1e-13
    assert h1.launch_count() > 0


@pytest.mark.parametrize("name", ["c2", "c3p4"])
def test_large_config_vcycle_and_cg(name):
    h, oh, _ = pair(name)
    for l in range(1, oh.L + 1):
        assert abs(h.get_eigen(l) - oh.levels[l].lam) <= 1e-10 * oh.levels[l].lam
    n = oh.leaf.n_free
    b = uniform_pm1(n)
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.vcycle(dev(b), x)
    assert rel(x.cpu().numpy(), mg.vcycle(oh, b)) < VC_TOL
    u = uniform_pm1(n, STREAM_PROBE)
    v = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.leaf_apply(dev(u), v)
    assert rel(v.cpu().numpy(), oh.A_leaf @ u) < OP_TOL
    bb = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, bb)
    xs = torch.zeros(n, device="cuda", dtype=torch.float64)
    it, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
    _, it_ref, _, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
    assert abs(it - it_ref) <= 1, (it, it_ref)


# ---------------------------------------------------------------- mixed precision
# SURVEY §8(f) row 1 / P:897: the V-cycle in fp32 inside the fp64 CG.
# The fp32 V-cycle is the fp64 one up to single-precision rounding: relative
# max-norm error bounded by a few hundred ulp(fp32) = 2^-24 per operation chain
# (MIXED_VC_TOL); CG keeps its fp64 residual and stopping test, so the iteration
# count stays within +-1 of the oracle's fp64 CG and the true residual <= 1e-8.
MIXED_VC_TOL = 2e-5
MIXED_CASES = [("c1", None), ("c3p2", None), ("c4", None, -1, C4S)]


@pytest.mark.parametrize("case", MIXED_CASES, ids=["c1", "c3p2", "c4s"])
def test_mixed_precision_vcycle_and_cg(case):
    name = case[0]
    cfg = dict(config(name))
    if len(case) > 2:
        cfg.update(case[3])
    coef = log_uniform_coef(4 ** cfg["dim"]) if cfg.get("coef") else None
    _, _, h = G.build_config(cfg, coef_level2=coef, mixed=True)
    _, oh, _ = pair(*case)
    for l in range(1, oh.L + 1):
        h.set_eigen(l, oh.levels[l].lam)
    n = oh.leaf.n_free
    b = uniform_pm1(n)
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.vcycle(dev(b), x)
    err = rel(x.cpu().numpy(), mg.vcycle(oh, b))
    assert 1e-9 < err < MIXED_VC_TOL, err          # fp32 rounding visible, bounded
    bb = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, bb)
    xs = torch.zeros(n, device="cuda", dtype=torch.float64)
    it, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
    _, it_ref, _, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
    assert abs(it - it_ref) <= 1, (it, it_ref)
    tr = np.linalg.norm(oh.b_leaf - oh.A_leaf @ xs.cpu().numpy()) / np.linalg.norm(oh.b_leaf)
    assert tr <= 1.01e-8


# ---------------------------------------------------------------- degenerate cases
# Edge cases of the method: a forest whose only level has no free DoF (every
# node on the Dirichlet boundary), a single free DoF, a sequence mesh with a
# long chain of nearly empty levels, and more ranks than leaves.
DEGENERATE = [("uniform", 2, 1, 1), ("uniform", 3, 1, 1), ("uniform", 2, 1, 2), ("quadrant", 2, 6, 1),
              ("circle", 3, 4, 2), ("quadrant", 2, 4, 1)]


@pytest.mark.parametrize("kind,d,L,k", DEGENERATE, ids=[f"{a}{b}d-L{c}-k{e}" for a, b, c, e in DEGENERATE])
def test_degenerate_forests(kind, d, L, k):
    f = G.gmg_forest_sequence(d, kind, L)
    part = G.gmg_partition(f, 1)
    h = G.gmg_setup(f, part, k=k)
    of = F.sequence(d, kind, L)
    oh = mg.build(of, k)
    n = oh.leaf.n_free
    assert h.info()["n_leaf_free"] == n
    for l in range(1, oh.L + 1):
        h.set_eigen(l, oh.levels[l].lam)
    b = uniform_pm1(n)
    x = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.vcycle(dev(b), x)
    if n:
        assert rel(x.cpu().numpy(), mg.vcycle(oh, b)) < VC_TOL
    bb = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, bb)
    xs = torch.zeros(n, device="cuda", dtype=torch.float64)
    it, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
    if n:
        _, it_ref, _, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
        assert abs(it - it_ref) <= 1, (it, it_ref)
    else:
        assert it == 0


def test_more_ranks_than_leaves_local_ranks():
    """p = 6 ranks on a 4-leaf forest: ranks without cells on some levels still
    take part in every exchange; the result equals one rank."""
    import threading
    f = G.gmg_forest_sequence(2, "uniform", 1)     # 4 leaves, one free Q2 DoF ring
    _, _, h1 = None, None, G.gmg_setup(f, G.gmg_partition(f, 1), k=2)
    n = h1.info()["n_leaf_free"]
    canon1 = h1.leaf_dofs()[3]
    b_can = uniform_pm1(n)
    x1 = torch.zeros(n, device="cuda", dtype=torch.float64)
    h1.vcycle(dev(b_can[canon1]), x1)
    ref = np.empty(n)
    ref[canon1] = x1.cpu().numpy()
    p = 6
    world = G.LocalWorld(p)
    part = G.gmg_partition(f, p)
    hs = [None] * p
    streams = [torch.cuda.Stream() for _ in range(p)]

    def setup(r):
        torch.cuda.set_device(0)
        hs[r] = G.gmg_setup(f, part, k=2, rank=r, comm=world)

    ts = [threading.Thread(target=setup, args=(r,)) for r in range(p)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    canon = hs[0].leaf_dofs()[3]
    res = [None] * p

    def work(r):
        torch.cuda.set_device(0)
        info = hs[r].info()
        fo, no = info["first_owned"], info["n_owned"]
        with torch.cuda.stream(streams[r]):
            bl = torch.tensor(b_can[canon[fo:fo + no]], device="cuda", dtype=torch.float64)
            xl = torch.zeros_like(bl)
            hs[r].vcycle(bl, xl, stream=streams[r].cuda_stream)
            streams[r].synchronize()
        res[r] = (fo, no, xl.cpu().numpy())

    ts = [threading.Thread(target=work, args=(r,)) for r in range(p)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    xv = np.empty(n)
    for fo, no, xl in res:
        xv[canon[fo:fo + no]] = xl
    assert rel(xv, ref) < 1e-13


# ---------------------------------------------------------------- random adaptive forests
# Seeded random refinement (a few leaves per pass, closed to 2:1 balance after each
# pass) in 2D/3D, Q1/Q2, one or two trees: every level operator, the V-cycle and
# the CG count against the oracle, fp64 and mixed precision.
RANDOM = [(2, 1, 11), (2, 2, 12), (3, 1, 13), (3, 2, 14), (3, 2, 15), (2, 2, 16)]


def _random_forest(d, seed, trees):
    rng = np.random.RandomState(seed)
    f = F.coarse_forest(d, trees)
    f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    for _ in range(6):
        m = np.zeros(f.n_leaves, dtype=bool)
        m[rng.randint(0, f.n_leaves, size=1 + f.n_leaves // 8)] = True
        f = F.close(F.refine(f, m))
        if f.n_leaves > (2500 if d == 2 else 1500):
            break
    return f


@pytest.mark.parametrize("d,k,seed", RANDOM, ids=[f"{d}d-k{k}-s{s}" for d, k, s in RANDOM])
def test_random_forest_vcycle_cg(d, k, seed):
    trees = [(0,) * d, (1,) + (0,) * (d - 1)] if seed % 2 == 0 else [(0,) * d]
    of = _random_forest(d, seed, trees)
    tree = of.tree_index()
    tpos = of.gc >> of.level[:, None]
    loc = of.gc - (tpos << of.level[:, None])
    lf = G.gmg_forest_create(d, [tuple(t) for t in of.trees], tree.astype(np.int32), of.level.astype(np.int8),
                             F.morton(loc, 32).astype(np.uint64))
    oh = mg.build(of, k)
    n = oh.leaf.n_free
    b = uniform_pm1(n, STREAM_PROBE, offset=seed)
    for mixed in (False, True):
        h = G.gmg_setup(lf, G.gmg_partition(lf, 1), k=k, mixed=mixed)
        if not mixed:
            for l, lev in enumerate(oh.levels):
                if lev.space.n == 0:
                    continue
                xv = uniform_pm1(lev.space.n, STREAM_PROBE, offset=100 * l)
                y = torch.zeros(lev.space.n, device="cuda", dtype=torch.float64)
                h.level_apply(l, dev(xv), y)
                assert rel(y.cpu().numpy(), lev.K @ xv) < OP_TOL, l
        for l in range(1, oh.L + 1):
            h.set_eigen(l, oh.levels[l].lam)
        x = torch.zeros(n, device="cuda", dtype=torch.float64)
        h.vcycle(dev(b), x)
        assert rel(x.cpu().numpy(), mg.vcycle(oh, b)) < (MIXED_VC_TOL if mixed else VC_TOL)
        bb = torch.zeros(n, device="cuda", dtype=torch.float64)
        h.rhs_constant(1.0, bb)
        xs = torch.zeros(n, device="cuda", dtype=torch.float64)
        it, relres, _ = h.solve_cg(bb, xs, rtol=1e-8)
        _, it_ref, _, _ = mg.pcg(oh, oh.b_leaf, rtol=1e-8)
        assert abs(it - it_ref) <= 1 and relres <= 1e-8, (mixed, it, it_ref)
