"""Config 5 at n = 1 (125.8M leaf DoFs, 11 levels) -- the bench headline -- at
its full size, in the launch configuration bench.py times (gmg_setup defaults:
CUDA graph, degree-4 Chebyshev, grandfamily + family operator kernels, the
fused residual + restriction, device order with R1).

Same checks as tests/test_full_size.py for configs 3 and 4, here on the forest
whose finest level runs 73 % of its families as grandfamily patches
(gfam_tensor_apply): (a) the level operator's output on sampled rows of the
finest level and of level 9 against the oracle's element matrix
(oracle/fem.py:element_laplace) summed over the cells of the
exported cell->DoF table; (b) properties that hold at any size: symmetry and
positivity of the level operator, R = P^T, symmetry, positivity and
linearity of the V-cycle, GMG-CG to 1e-8."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config_c5, uniform_pm1, STREAM_PROBE  # noqa: E402
from oracle import fem  # noqa: E402

OP_TOL = 1e-12
VC_TOL = 1e-10
N_SAMPLE = 4096


def dev(a):
    return torch.tensor(np.asarray(a), device="cuda", dtype=torch.float64)


def dot(a, b):
    return float(torch.dot(a, b))


@pytest.fixture(scope="module")
def h5():
    _, _, h = G.build_config(config_c5(1))
    yield h
    del h
    torch.cuda.empty_cache()


@pytest.mark.parametrize("which", ["finest", "level9"])
def test_c5_level_apply_sampled_rows(h5, which):
    info = h5.info()
    L = info["n_levels"] - 1
    l = L if which == "finest" else L - 1
    n = info["level_dofs"][l]
    x = uniform_pm1(n, STREAM_PROBE, offset=29)
    y = torch.zeros(n, device="cuda", dtype=torch.float64)
    h5.level_apply(l, dev(x), y)
    y = y.cpu().numpy()
    cd = h5.cell_dofs(l)
    rows = np.random.default_rng(190403317 + 5 * l).choice(n, size=min(N_SAMPLE, n), replace=False)
    Ke = fem.element_laplace(info["dim"], info["k"], 2.0 ** -l)
    cells, bs = np.nonzero(np.isin(cd, rows))
    cdr = cd[cells]
    del cd
    xc = np.where(cdr >= 0, x[np.maximum(cdr, 0)], 0.0)
    contrib = np.einsum("ij,ij->i", Ke[bs], xc)
    ref = np.zeros(n)
    np.add.at(ref, cdr[np.arange(len(cells)), bs], contrib)
    scale = np.abs(ref[rows]).max()
    assert scale > 0
    err = np.abs(y[rows] - ref[rows]).max() / scale
    assert err < OP_TOL, (l, err)


def test_c5_level_operator_symmetric_positive(h5):
    info = h5.info()
    L = info["n_levels"] - 1
    n = info["level_dofs"][L]
    x, z = dev(uniform_pm1(n, STREAM_PROBE, offset=31)), dev(uniform_pm1(n, STREAM_PROBE, offset=37))
    kx, kz = torch.zeros_like(x), torch.zeros_like(z)
    h5.level_apply(L, x, kx)
    h5.level_apply(L, z, kz)
    a, b = dot(kx, z), dot(x, kz)
    assert abs(a - b) <= OP_TOL * float(kx.norm() * z.norm())
    assert dot(x, kx) > 0 and dot(z, kz) > 0


def test_c5_transfers_adjoint(h5):
    info = h5.info()
    L = info["n_levels"] - 1
    nf, nc = info["level_dofs"][L], info["level_dofs"][L - 1]
    xc = dev(uniform_pm1(nc, STREAM_PROBE, offset=41))
    rf = dev(uniform_pm1(nf, STREAM_PROBE, offset=43))
    xf = torch.zeros(nf, device="cuda", dtype=torch.float64)
    dc = torch.zeros(nc, device="cuda", dtype=torch.float64)
    h5.prolongate(L, xc, xf)
    h5.restrict(L, rf, dc)
    assert abs(dot(dc, xc) - dot(rf, xf)) <= OP_TOL * float(dc.norm() * xc.norm())


def test_c5_vcycle_symmetric_positive_linear(h5):
    n = h5.info()["n_leaf_free"]
    b1, b2 = dev(uniform_pm1(n)), dev(uniform_pm1(n, STREAM_PROBE))
    v1, v2, v3 = torch.zeros_like(b1), torch.zeros_like(b1), torch.zeros_like(b1)
    h5.vcycle(b1, v1)
    h5.vcycle(b2, v2)
    assert abs(dot(v1, b2) - dot(b1, v2)) <= VC_TOL * float(v1.norm() * b2.norm())
    assert dot(v1, b1) > 0 and dot(v2, b2) > 0
    h5.vcycle(2.5 * b1, v3)
    assert float((v3 - 2.5 * v1).abs().max()) <= 1e-13 * float(v3.abs().max())


def test_c5_cg_converges(h5):
    n = h5.info()["n_leaf_free"]
    b = torch.zeros(n, device="cuda", dtype=torch.float64)
    h5.rhs_constant(1.0, b)
    x = torch.zeros_like(b)
    it, relres, _ = h5.solve_cg(b, x, rtol=1e-8)
    assert relres <= 1e-8 and 1 <= it <= 12, (it, relres)
    r = torch.zeros_like(b)
    h5.leaf_apply(x, r)
    assert float((b - r).norm() / b.norm()) <= 1.01e-8
