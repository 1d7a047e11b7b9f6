"""Pins of the oracle's spaces, operators, transfers, smoother, V-cycle and CG
(no GPU).  Each test checks the oracle against something other than itself:
textbook closed forms, exact polynomial reproduction, Galerkin identities,
the dense literal algorithm of oracle.abstract, or known eigenvalues."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import forest as F, fem, mg, abstract
from oracle.spaces import Lattice
from gmg_inputs import config, uniform_pm1

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def uniform(d, L, trees=None):
    f = F.coarse_forest(d, trees or [(0,) * d])
    for _ in range(L):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    return f


def small_adaptive(d, seed_cells, base=2):
    f = uniform(d, base)
    for p in seed_cells:
        m = np.zeros(f.n_leaves, dtype=bool)
        m[p % f.n_leaves] = True
        f = F.close(F.refine(f, m))
    return f


# ------------------------------------------------------------- 1-D matrices
def test_1d_closed_forms():
    """Textbook Q1/Q2 stiffness and mass matrices (exact rationals) vs the
    oracle's Gauss-quadrature derivation from the Lagrange basis."""
    K1, M1 = fem.matrices_1d(1)
    assert np.allclose(K1, [[1, -1], [-1, 1]], atol=1e-15)
    assert np.allclose(M1, [[1 / 3, 1 / 6], [1 / 6, 1 / 3]], atol=1e-15)
    K2, M2 = fem.matrices_1d(2)
    assert np.allclose(K2, np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / 3, atol=1e-14)
    assert np.allclose(M2, np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30, atol=1e-15)
    assert np.allclose(fem.mass_weights_1d(2), [1 / 6, 2 / 3, 1 / 6], atol=1e-15)
    # sub-interval matrices add up (config 4 sub-box integration)
    for k in (1, 2):
        Ks = sum(fem.matrices_1d(k, s / 4, (s + 1) / 4)[0] for s in range(4))
        Ms = sum(fem.matrices_1d(k, s / 4, (s + 1) / 4)[1] for s in range(4))
        K, M = fem.matrices_1d(k)
        assert np.allclose(Ks, K, atol=1e-13) and np.allclose(Ms, M, atol=1e-14)


def test_embedding_values():
    # Q2 child embeddings E0 / E1 (SURVEY c.1 step 7) and Q1 centre weight 1/4
    E0 = fem.lagrange(2, np.array([0, 0.25, 0.5]))
    E1 = fem.lagrange(2, np.array([0.5, 0.75, 1.0]))
    assert np.allclose(E0, [[1, 0, 0], [3 / 8, 3 / 4, -1 / 8], [0, 1, 0]], atol=1e-15)
    assert np.allclose(E1, [[0, 1, 0], [-1 / 8, 3 / 4, 3 / 8], [0, 0, 1]], atol=1e-15)
    w = np.kron(fem.lagrange(1, np.array([0.5])), fem.lagrange(1, np.array([0.5])))
    assert np.allclose(w, 0.25)


def test_element_matrix_properties():
    for d in (2, 3):
        for k in (1, 2):
            A = fem.element_laplace(d, k, 2.0 ** -3)
            assert np.allclose(A, A.T, atol=0)
            assert np.allclose(A.sum(axis=1), 0, atol=1e-13)       # Laplace kills constants
    A = fem.element_laplace(2, 1, 0.37)
    assert np.allclose(np.diag(A), 2 / 3)                           # S:280, h-independent in 2D


# ------------------------------------------------------------- config 1 structure
def test_config1_level_structure():
    g = json.load(open(os.path.join(GOLD, "config_counts.json")))["c1"]
    f = F.generate(config("c1"))
    h = mg.build(f, 1, eig=False)
    for l, lev in enumerate(h.levels):
        s = lev.space
        row = [len(s.cells.gc), s.n + s.n_boundary, s.n_boundary, int(lev.E.sum()),
               int(lev.S.sum()), int(s.cells.is_leaf.sum())]
        assert row == g["per_level"][l]
    lf = h.leaf
    assert lf.X.shape[0] == g["leaf_nodes"] and lf.n_free == g["free"]
    assert int(lf.hanging.sum()) == g["hanging"] and int(lf.dirichlet.sum()) == g["dirichlet"]


def test_lambda_rule():
    """lambda(n) in {m, m-1}, m = max level of the leaves having n as a node."""
    f = F.generate(config("c1"))
    h = mg.build(f, 1, eig=False)
    lf = h.leaf
    nn = lf.cell_nodes.shape[1]
    mx = np.full(lf.X.shape[0], -1)
    mn = np.full(lf.X.shape[0], 99)
    np.maximum.at(mx, lf.cell_nodes.ravel(), np.repeat(f.level, nn))
    np.minimum.at(mn, lf.cell_nodes.ravel(), np.repeat(f.level, nn))
    free = lf.free_index >= 0
    lam = lf.lam
    m = mx[free]
    assert np.all((lam == m) | (lam == m - 1))
    assert np.all(lam[mn[free] == m] == m[mn[free] == m])


# ------------------------------------------------------------- operators
@pytest.mark.parametrize("d,k", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_level_operators_spd_and_galerkin(d, k):
    f = uniform(d, 3 if d == 2 else 2)
    h = mg.build(f, k, eig=False)
    for l, lev in enumerate(h.levels):
        K = lev.K.toarray()
        if K.size == 0:
            continue
        assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()   # up to summation order
        if lev.S.any():
            AS = K[np.ix_(lev.S, lev.S)]
            np.linalg.cholesky(AS)
        if l > 0:
            P = lev.P.toarray()
            # Galerkin A_{l-1} = P^T A_l P on nested uniform levels (all rows S)
            G = P.T @ K @ P
            assert np.allclose(G, h.levels[l - 1].K.toarray(), atol=1e-12 * np.abs(K).max())


def test_galerkin_variable_coefficient_subbox():
    """Config-4 style coefficient per level-2 cell; levels 0-1 integrate it over
    their sub-boxes, so A_l = P^T A_{l+1} P must hold on every uniform level
    (the level forms are restrictions of a(.,.))."""
    for d, k in [(2, 2), (3, 1), (3, 2)]:
        f = uniform(d, 3)
        ncoef = (1 << (2 * d))
        coefs = np.power(10.0, 4 * np.linspace(0.05, 0.95, ncoef) - 2)[np.random.RandomState(1).permutation(ncoef)]
        h = mg.build(f, k, coef_level2=coefs, eig=False)
        for l in range(1, h.L + 1):
            K = h.levels[l].K
            P = h.levels[l].P
            G = (P.T @ K @ P).toarray()
            Kc = h.levels[l - 1].K.toarray()
            if Kc.size:
                assert np.allclose(G, Kc, atol=1e-12 * np.abs(Kc).max())


def test_transfer_polynomial_exactness():
    """P reproduces Q_k functions: interpolant of a coarse Q2 polynomial that
    vanishes on the boundary is mapped to its fine interpolant."""
    f = small_adaptive(2, [0, 5, 17])
    h = mg.build(f, 2, eig=False)
    u = lambda X: (X[:, 0] * (1 - X[:, 0])) * (X[:, 1] * (1 - X[:, 1]))
    for l in range(1, h.L + 1):
        fine = h.levels[l].space
        coarse = h.levels[l - 1].space
        xf = u(fine.X / float(h.lat.T))
        xc = u(coarse.X / float(h.lat.T))
        assert np.allclose(h.levels[l].P @ xc, xf, atol=1e-13)


def test_q1_partition_of_unity_interior():
    f = uniform(2, 3)
    h = mg.build(f, 1, eig=False)
    P = h.levels[3].P
    X = h.levels[3].space.X / float(h.lat.T)
    inner = np.all((X > 0.25) & (X < 0.75), axis=1)
    assert np.allclose((P @ np.ones(P.shape[1]))[inner], 1.0)


# ------------------------------------------------------------- leaf system
@pytest.mark.parametrize("d", [2, 3])
def test_q2_reproduces_quadratic_with_hanging_nodes(d):
    """u = prod x_i(1 - x_i) lies in Q2 even with hanging nodes, so the discrete
    solution equals its interpolant exactly (Galerkin orthogonality)."""
    f = small_adaptive(d, [0, 3, 11] if d == 2 else [0, 9], base=2 if d == 2 else 1)
    h = mg.build(f, 2, eig=False)
    assert h.leaf.hanging.any()
    def u(X):
        return np.prod(X * (1 - X), axis=1)
    def mlap(X):
        s = np.zeros(X.shape[0])
        for i in range(d):
            s += 2 * np.prod(np.delete(X * (1 - X), i, axis=1), axis=1)
        return s
    A, b = fem.leaf_system(f, h.leaf, h.lat, None, rhs=mlap)
    x = spla.spsolve(A.tocsc(), b)
    ui = fem.interpolate_leaf(h.leaf, h.lat, u)
    assert np.allclose(x, ui, atol=1e-12)


@pytest.mark.parametrize("k,rate", [(1, 2.0), (2, 3.0)])
def test_l2_convergence_rate(k, rate):
    errs = []
    hs = []
    u = lambda X: np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1])
    rhs = lambda X: 2 * np.pi ** 2 * u(X)
    for L in (3, 4, 5):
        f = uniform(2, L)
        h = mg.build(f, k, eig=False)
        A, b = fem.leaf_system(f, h.leaf, h.lat, None, rhs=rhs)
        x = spla.spsolve(A.tocsc(), b)
        errs.append(fem.l2_error(f, h.leaf, h.lat, x, u))
        hs.append(2.0 ** -L)
    slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
    assert abs(slope - rate) < 0.1


def test_leaf_matrix_spd_symmetric():
    f = F.generate(config("c1"))
    h = mg.build(f, 1, eig=False)
    A = h.A_leaf
    assert abs(A - A.T).max() == 0
    ev = np.linalg.eigvalsh(A.toarray())
    assert ev.min() > 0


# ------------------------------------------------------------- eigen / chebyshev
def test_eigen_estimate_closed_form_q1():
    """Uniform Q1 2D: lambda(D^-1 A) = 1 + cos^2(pi/n)/2 (closed form, SURVEY c.3).
    Exact when n_S <= 10 (Krylov space exhausted), otherwise a Ritz lower bound."""
    f = uniform(2, 5)
    h = mg.build(f, 1)
    for l in range(2, 6):
        n = 1 << l
        true = 1 + 0.5 * np.cos(np.pi / n) ** 2
        est = h.levels[l].lam
        nS = int(h.levels[l].S.sum())
        if nS <= 10:
            assert abs(est - true) < 1e-12
        else:
            assert est <= true * (1 + 1e-12) and est >= 0.95 * true
    assert abs(h.levels[2].lam - 1.25) < 1e-13


def test_eigen_rhs_pattern():
    f = uniform(2, 4)
    h = mg.build(f, 1, eig=False)
    v = mg.eigen_rhs(h.levels[4])
    vs = v[h.levels[4].S]
    assert np.allclose(vs[:12], np.arange(-5.5, 6.0, 1.0))
    assert vs[12] == -5.5


def test_chebyshev_recurrence_equals_Tm_propagator():
    f = small_adaptive(2, [0, 7])
    h = mg.build(f, 2)
    rs = np.random.RandomState(0)
    for l in range(1, h.L + 1):
        lev = h.levels[l]
        S = lev.S
        AS = lev.K.toarray()[np.ix_(S, S)]
        g = rs.randn(lev.space.n) * lev.S
        x0 = rs.randn(lev.space.n) * lev.S
        for deg in (1, 2, 4, 5):
            x = mg.chebyshev(lev, g, x0, deg)
            ref = abstract.cheb_smooth_dense(AS, g[S], x0[S], lev.lam, deg)
            assert np.allclose(x[S], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


# ------------------------------------------------------------- V-cycle
def _abstract_vs_oracle(f, k, b=None):
    h = mg.build(f, k)
    am = abstract.AbstractMG(f, k, [lev.lam for lev in h.levels], degree=h.degree)
    lat = h.lat
    keys = np.array(am.leaf_keys())
    lk = lat.lin(h.leaf.X[h.leaf.free_index >= 0])
    ak = lat.lin(keys)
    o = np.argsort(lk)
    perm = o[np.searchsorted(lk[o], ak)]
    assert np.all(lk[perm] == ak)
    assert np.allclose(am.A[-1], h.A_leaf.toarray()[np.ix_(perm, perm)], atol=1e-13)
    if b is None:
        b = uniform_pm1(h.leaf.n_free)
    x1 = mg.vcycle(h, b)
    x2 = am.vcycle(am.L, b[perm])
    return np.abs(x1[perm] - x2).max() / np.abs(x2).max()


def test_vcycle_equals_abstract_config1():
    f = F.generate(config("c1"))
    assert _abstract_vs_oracle(f, 1) < 1e-13


@pytest.mark.parametrize("d,k,cells", [(2, 2, [0, 5, 9]), (3, 1, [0, 20]), (3, 2, [3]),
                                       (2, 1, [12, 13, 40, 41])])
def test_vcycle_equals_abstract_adaptive(d, k, cells):
    f = small_adaptive(d, cells, base=2 if d == 2 else 1)
    assert _abstract_vs_oracle(f, k) < 1e-12


def test_vcycle_equals_abstract_lshape():
    cfg = dict(config("c2"))
    cfg["lmax"] = 5
    cfg["s"] = 0
    cfg["global_refinements"] = 1
    f = F.generate(cfg)
    assert _abstract_vs_oracle(f, 2) < 1e-12


def test_vcycle_uniform_is_textbook():
    # no refinement edge anywhere: every level DoF is S
    f = uniform(2, 4)
    h = mg.build(f, 2)
    assert all(not lev.E.any() for lev in h.levels)
    assert _abstract_vs_oracle(f, 2) < 1e-13


def test_vcycle_linear_symmetric_spd():
    f = F.generate(config("c1"))
    h = mg.build(f, 1)
    rs = np.random.RandomState(3)
    n = h.leaf.n_free
    assert np.all(mg.vcycle(h, np.zeros(n)) == 0)
    for _ in range(5):
        v, w = rs.randn(n), rs.randn(n)
        Mv, Mw = mg.vcycle(h, v), mg.vcycle(h, w)
        scale = np.linalg.norm(v) * np.linalg.norm(w) * max(np.abs(Mv).max(), 1e-300) / max(np.abs(v).max(), 1e-300)
        assert abs(v @ Mw - w @ Mv) <= 1e-12 * scale
        assert v @ Mv > 0
        a, c = 0.7, -1.3
        assert np.allclose(mg.vcycle(h, a * v + c * w), a * Mv + c * Mw, atol=1e-12 * np.abs(Mv).max())


# ------------------------------------------------------------- CG
def test_cg_exact_termination_small():
    f = uniform(2, 1)
    h = mg.build(f, 1)
    assert h.leaf.n_free == 1
    x, it, rel, _ = mg.pcg(h, h.b_leaf, precond=lambda r: r)
    assert it == 1 and rel < 1e-14


def test_cg_mesh_independent():
    its = []
    for L in (3, 4, 5, 6):
        f = uniform(2, L)
        h = mg.build(f, 2)
        _, it, rel, _ = mg.pcg(h, h.b_leaf, rtol=1e-8)
        assert rel <= 1e-8
        its.append(it)
    assert max(its) - min(its) <= 2


def test_cg_config1_true_residual():
    f = F.generate(config("c1"))
    h = mg.build(f, 1)
    x, it, rel, _ = mg.pcg(h, h.b_leaf, rtol=1e-8)
    tr = np.linalg.norm(h.b_leaf - h.A_leaf @ x) / np.linalg.norm(h.b_leaf)
    assert tr <= 1e-8 and it < 20
