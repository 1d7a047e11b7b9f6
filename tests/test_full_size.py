"""Configs 3 (49.8M leaf DoFs, 11 levels) and 4 (107M leaf nodes, 20 levels,
variable coefficient) at their full sizes, in the launch configuration bench.py times (gmg_setup defaults: CUDA graph, degree-4
Chebyshev, family-tensor operator kernels, device order with R1).

The oracle cannot assemble this hierarchy in seconds, so the checks are
(a) sampled rows: the level operator's output on 4096 random rows against the
    oracle's element matrix (oracle/fem.py:element_laplace) summed
    over the cells of the exported cell->DoF table, row by row (the integer
    topology itself is pinned bit-exact against the oracle on small forests in
    test_parity_integer.py and by the config-3 level counts in test_sequences.py);
(b) properties that hold at any size: symmetry and positivity of the level
    operator, R = P^T, symmetry, positivity and linearity of the
    V-cycle as a preconditioner (it is a symmetric operator because pre- and
    post-smoother are the same Chebyshev polynomial; the oracle V-cycle is
    symmetric to 1e-15 on config 1), GMG-CG convergence to 1e-8, and the mixed
    precision V-cycle within MIXED_VC_TOL of the fp64 one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, uniform_pm1, log_uniform_coef, STREAM_PROBE  # noqa: E402
from oracle import fem  # noqa: E402

OP_TOL = 1e-12
VC_TOL = 1e-10
MIXED_VC_TOL = 2e-5
N_SAMPLE = 4096

_h = {}


def hier(mixed=False):
    if mixed not in _h:
        _, _, h = G.build_config(config("c3"), mixed=mixed)
        _h[mixed] = h
    return _h[mixed]


def dev(a):
    return torch.tensor(np.asarray(a), device="cuda", dtype=torch.float64)


def dot(a, b):
    return float(torch.dot(a, b))


@pytest.fixture(scope="module")
def h64():
    return hier(False)


@pytest.mark.parametrize("which", ["finest", "middle"])
def test_c3_level_apply_sampled_rows(h64, which):
    info = h64.info()
    L = info["n_levels"] - 1
    l = L if which == "finest" else L // 2
    n = info["level_dofs"][l]
    x = uniform_pm1(n, STREAM_PROBE, offset=17)
    y = torch.zeros(n, device="cuda", dtype=torch.float64)
    h64.level_apply(l, dev(x), y)
    y = y.cpu().numpy()
    # oracle rows: sum over the level-l cells containing the row's node of Ke[b, :] x[cell]
    cd = h64.cell_dofs(l)
    rows = np.random.default_rng(190403317 + l).choice(n, size=min(N_SAMPLE, n), replace=False)
    Ke = fem.element_laplace(info["dim"], info["k"], 2.0 ** -l)
    hit = np.isin(cd, rows)
    cells, bs = np.nonzero(hit)
    xc = np.where(cd[cells] >= 0, x[np.maximum(cd[cells], 0)], 0.0)     # x on those cells
    contrib = np.einsum("ij,ij->i", Ke[bs], xc)
    ref = np.zeros(n)
    np.add.at(ref, cd[cells, bs], contrib)
    scale = np.abs(ref[rows]).max()
    assert scale > 0
    err = np.abs(y[rows] - ref[rows]).max() / scale
    assert err < OP_TOL, (l, err)


def test_c3_level_operator_symmetric_positive(h64):
    info = h64.info()
    L = info["n_levels"] - 1
    n = info["level_dofs"][L]
    x, z = dev(uniform_pm1(n, STREAM_PROBE, offset=1)), dev(uniform_pm1(n, STREAM_PROBE, offset=2))
    kx, kz = torch.zeros_like(x), torch.zeros_like(z)
    h64.level_apply(L, x, kx)
    h64.level_apply(L, z, kz)
    a, b = dot(kx, z), dot(x, kz)
    assert abs(a - b) <= OP_TOL * float(kx.norm() * z.norm())
    assert dot(x, kx) > 0 and dot(z, kz) > 0


def test_c3_transfers_adjoint(h64):
    info = h64.info()
    L = info["n_levels"] - 1
    nf, nc = info["level_dofs"][L], info["level_dofs"][L - 1]
    xc = dev(uniform_pm1(nc, STREAM_PROBE, offset=3))
    rf = dev(uniform_pm1(nf, STREAM_PROBE, offset=4))
    xf = torch.zeros(nf, device="cuda", dtype=torch.float64)
    dc = torch.zeros(nc, device="cuda", dtype=torch.float64)
    h64.prolongate(L, xc, xf)
    h64.restrict(L, rf, dc)
    lhs, rhs = dot(dc, xc), dot(rf, xf)
    assert abs(lhs - rhs) <= OP_TOL * float(dc.norm() * xc.norm())


def test_c3_vcycle_symmetric_positive_linear(h64):
    n = h64.info()["n_leaf_free"]
    b1, b2 = dev(uniform_pm1(n)), dev(uniform_pm1(n, STREAM_PROBE))
    v1, v2, v3 = torch.zeros_like(b1), torch.zeros_like(b1), torch.zeros_like(b1)
    h64.vcycle(b1, v1)
    h64.vcycle(b2, v2)
    a, b = dot(v1, b2), dot(b1, v2)
    assert abs(a - b) <= VC_TOL * float(v1.norm() * b2.norm())
    assert dot(v1, b1) > 0 and dot(v2, b2) > 0
    h64.vcycle(2.5 * b1, v3)
    assert float((v3 - 2.5 * v1).abs().max()) <= 1e-13 * float(v3.abs().max())


def test_c3_cg_converges(h64):
    n = h64.info()["n_leaf_free"]
    b = torch.zeros(n, device="cuda", dtype=torch.float64)
    h64.rhs_constant(1.0, b)
    x = torch.zeros_like(b)
    it, relres, _ = h64.solve_cg(b, x, rtol=1e-8)
    assert relres <= 1e-8 and 1 <= it <= 12, (it, relres)
    r = torch.zeros_like(b)
    h64.leaf_apply(x, r)
    assert float((b - r).norm() / b.norm()) <= 1.01e-8


def test_c3_mixed_precision_vcycle(h64):
    hm = hier(True)
    n = h64.info()["n_leaf_free"]
    b = dev(uniform_pm1(n))
    x64, x32 = torch.zeros_like(b), torch.zeros_like(b)
    h64.vcycle(b, x64)
    hm.vcycle(b, x32)
    err = float((x32 - x64).abs().max() / x64.abs().max())
    assert 1e-9 < err < MIXED_VC_TOL, err


# ---------------------------------------------------------------- config 4, full size
# 107M leaf nodes, 20 levels, a log-uniform per level-2 cell (R15, R20): sampled
# rows of the level operator on a coefficient level against a(cell) times the
# oracle element matrix, and the preconditioner / CG properties.
_h4 = {}


def hier4():
    if "h" not in _h4:
        cfg = config("c4")
        coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"]))
        f = G.gmg_forest_generate(G.recipe_from_config(cfg))
        part = G.gmg_partition(f, 1)
        _h4["h"] = (G.gmg_setup(f, part, k=cfg["k"], coef_level2=coef), part, coef)
    return _h4["h"]


@pytest.mark.parametrize("which", ["finest", "middle"])
def test_c4_level_apply_sampled_rows(which):
    h, part, coef = hier4()
    info = h.info()
    L = info["n_levels"] - 1
    l = L if which == "finest" else 10
    n = info["level_dofs"][l]
    x = uniform_pm1(n, STREAM_PROBE, offset=23)
    y = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.level_apply(l, dev(x), y)
    y = y.cpu().numpy()
    cd = h.cell_dofs(l)
    keys, _, _ = part.level_cells(l)
    keys2, _, _ = part.level_cells(2)
    a_cell = coef[np.searchsorted(keys2, keys >> np.uint64(3 * (l - 2)))]   # R15: the level-2 ancestor's a
    rows = np.random.default_rng(190403317 + l).choice(n, size=min(N_SAMPLE, n), replace=False)
    Ke = fem.element_laplace(info["dim"], info["k"], 2.0 ** -l)
    cells, bs = np.nonzero(np.isin(cd, rows))
    xc = np.where(cd[cells] >= 0, x[np.maximum(cd[cells], 0)], 0.0)
    contrib = a_cell[cells] * np.einsum("ij,ij->i", Ke[bs], xc)
    ref = np.zeros(n)
    np.add.at(ref, cd[cells, bs], contrib)
    err = np.abs(y[rows] - ref[rows]).max() / np.abs(ref[rows]).max()
    assert err < OP_TOL, (l, err)


def test_c4_vcycle_symmetric_and_cg():
    h, _, _ = hier4()
    n = h.info()["n_leaf_free"]
    b1, b2 = dev(uniform_pm1(n)), dev(uniform_pm1(n, STREAM_PROBE))
    v1, v2 = torch.zeros_like(b1), torch.zeros_like(b1)
    h.vcycle(b1, v1)
    h.vcycle(b2, v2)
    assert abs(dot(v1, b2) - dot(b1, v2)) <= VC_TOL * float(v1.norm() * b2.norm())
    assert dot(v1, b1) > 0 and dot(v2, b2) > 0
    b = torch.zeros(n, device="cuda", dtype=torch.float64)
    h.rhs_constant(1.0, b)
    x = torch.zeros_like(b)
    it, relres, _ = h.solve_cg(b, x, rtol=1e-8)
    assert relres <= 1e-8 and 1 <= it <= 15, (it, relres)
    r = torch.zeros_like(b)
    h.leaf_apply(x, r)
    assert float((b - r).norm() / b.norm()) <= 1.01e-8
