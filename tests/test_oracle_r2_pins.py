"""Oracle pins added in round 2 (VERDICT r1 "What's missing" #4, "What's weak" #1).

Each test checks the oracle against something other than itself:

* the level-DoF owner rule (R25) and the per-level partition (R29)
  against hand-derived values (tests/golden/owner_rules.json) and against a
  brute-force plain-loop evaluation of the definitions that imports none of
  the oracle's partition or space helpers;
* the literal two-level cycle against its dense closed form: with dense
  direct solves and the Chebyshev error propagator E_m = T_m((theta - D^-1 A)
  / delta) / T_m(theta / delta) evaluated through an eigendecomposition (not the
  three-term recurrence), u1 = G d, u2 = u1 + P A_0^-1 P^T (d - A u1),
  u3 = u2 + G (d - A u2), G = (I - E_m) A^-1 (the V-cycle
  with two levels), and the same with local smoothing on an adaptive two-level
  mesh where the residual carries the edge rows and the post-smoother the edge
  term (Section 2.3);
* SPD of the smoothed block A_l^SS on adaptive levels and the Neumann kernel
  (constants) of the element matrices and of the assembled level operator
  including Dirichlet nodes (PAPER.md:140-155 weak form; every element matrix
  of a Laplacian annihilates constants).
"""
import json
import os
from itertools import product

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

from oracle import forest as F, fem, mg, partition as Pt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _uniform2d(L):
    f = F.coarse_forest(2, [(0, 0)])
    for _ in range(L):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    return f


def _owner_by_X(space):
    return {tuple(int(v) for v in x): int(o) for x, o in zip(space.X, space.owner)}


# ------------------------------------------------------------------ owner rule: golden
@pytest.mark.parametrize("case", ["first_child_p4", "first_child_p3"])
def test_owner_rule_hand_derived(case):
    g = json.load(open(os.path.join(GOLD, "owner_rules.json")))[case]
    p = g["n_ranks"]
    f = _uniform2d(2)
    assert Pt.leaf_owners(f, p).tolist() == g["leaf_owner_by_sfc_index"]
    cells = Pt.level_cells(f, Pt.leaf_owners(f, p))
    assert cells[1].owner.tolist() == g["level1_cell_owner_by_morton"]
    T = mg.topology(f, 1, p)
    got2 = _owner_by_X(T.spaces[2])
    want2 = {tuple(int(v) for v in k.split(",")): o for k, o in g["level2_dof_owner"].items()}
    assert got2 == want2
    if "level1_dof_owner" in g:
        want1 = {tuple(int(v) for v in k.split(",")): o for k, o in g["level1_dof_owner"].items()}
        assert _owner_by_X(T.spaces[1]) == want1
    assert T.spaces[0].n == 0 or set(T.spaces[0].owner.tolist()) == {0}


def test_per_level_owners_hand_derived():
    g = json.load(open(os.path.join(GOLD, "owner_rules.json")))["per_level_p3"]
    f = _uniform2d(2)
    cells = Pt.per_level_owners(Pt.level_cells(f, Pt.leaf_owners(f, 3)), 3)
    assert cells[0].owner.tolist() == g["level0_cell_owner"]
    assert cells[1].owner.tolist() == g["level1_cell_owner_by_morton"]
    assert cells[2].owner.tolist() == g["level2_cell_owner_by_sfc_index"]


# ------------------------------------------------------------------ owner rule: brute force
def _brute_force_owners(f, k, p):
    """The definitions as plain loops over leaves, cells and nodes (no oracle
    partition/space helpers): R4 intervals, first SFC leaf of a subtree (=
    recursive first-child rule), node owner = min over the level-l cells
    having the node of their parent's owner, level 0 -> rank 0 (R25)."""
    n = f.n_leaves
    base, rem = divmod(n, p)
    leaf_owner, r, left = [], 0, base + (1 if rem > 0 else 0)
    for i in range(n):
        while left == 0:
            r += 1
            left = base + (1 if r < rem else 0)
        leaf_owner.append(r)
        left -= 1
    cell_owner = {}                              # (level, gc tuple) -> owner
    for i in range(n):                           # leaves in SFC order
        lv = int(f.level[i])
        for l in range(lv + 1):
            key = (l, tuple(int(c) >> (lv - l) for c in f.gc[i]))
            if key not in cell_owner:            # first leaf of the subtree
                cell_owner[key] = leaf_owner[i]
    L = f.max_level
    d = f.dim
    node_owner = [dict() for _ in range(L + 1)]
    for (l, gc), _ in cell_owner.items():
        comp = 0 if l == 0 else cell_owner[(l - 1, tuple(c >> 1 for c in gc))]
        for a in product(range(k + 1), repeat=d):
            X = tuple((k * gc[j] + a[j]) << (L - l) for j in range(d))
            node_owner[l][X] = min(node_owner[l].get(X, p), comp)
    return leaf_owner, cell_owner, node_owner


def _random_forest(dim, seed, base, steps):
    rng = np.random.default_rng(seed)
    f = F.coarse_forest(dim, [(0,) * dim] if dim == 3 else [(0, 0), (1, 0)])
    for _ in range(base):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    for _ in range(steps):
        m = rng.random(f.n_leaves) < 0.15
        f = F.close(F.refine(f, m))
    return f


@pytest.mark.parametrize("dim,k,p,seed", [(2, 1, 3, 1), (2, 2, 5, 2), (2, 1, 7, 3), (3, 1, 4, 4), (3, 2, 3, 5)])
def test_owner_rule_brute_force(dim, k, p, seed):
    f = _random_forest(dim, seed, base=2, steps=2)
    leaf_owner, cell_owner, node_owner = _brute_force_owners(f, k, p)
    assert Pt.leaf_owners(f, p).tolist() == leaf_owner
    cells = Pt.level_cells(f, Pt.leaf_owners(f, p))
    for l, lc in enumerate(cells):
        for gc, o in zip(lc.gc, lc.owner):
            assert cell_owner[(l, tuple(int(c) for c in gc))] == int(o)
    T = mg.topology(f, k, p)
    checked = 0
    for l, s in enumerate(T.spaces):
        got = _owner_by_X(s)
        for X, o in got.items():
            want = 0 if l == 0 else node_owner[l][X]
            assert o == want, (l, X, o, want)
            checked += 1
    assert checked > 50
    # invariant of the rule: each owned DoF lies in a family its owner computes
    for l in range(1, len(T.spaces)):
        comp_nodes = {}
        for (lv, gc), _ in cell_owner.items():
            if lv != l:
                continue
            q = cell_owner[(l - 1, tuple(c >> 1 for c in gc))]
            for a in product(range(k + 1), repeat=dim):
                X = tuple((k * gc[j] + a[j]) << (f.max_level - l) for j in range(dim))
                comp_nodes.setdefault(X, set()).add(q)
        for X, o in _owner_by_X(T.spaces[l]).items():
            assert o in comp_nodes[X]


@pytest.mark.parametrize("dim,p,seed", [(2, 3, 7), (2, 6, 8), (3, 4, 9)])
def test_per_level_owners_properties(dim, p, seed):
    """R29 on random adaptive forests: families (cells with a common parent) are
    never split, owners are non-decreasing along the SFC, and every rank's cell
    count on a level is within one family (2^d cells) of N_l/p."""
    f = _random_forest(dim, seed, base=2 if dim == 2 else 1, steps=2)
    cells = Pt.per_level_owners(Pt.level_cells(f, Pt.leaf_owners(f, p)), p)
    for l, lc in enumerate(cells):
        own = lc.owner
        assert np.all(np.diff(own) >= 0)
        if l > 0:
            fam = {}
            for gc, o in zip(lc.gc, own):
                fam.setdefault(tuple(int(c) >> 1 for c in gc), set()).add(int(o))
            assert all(len(v) == 1 for v in fam.values())
        n = lc.gc.shape[0]
        cnt = np.bincount(own, minlength=p)
        if l > 0:
            assert np.all(np.abs(cnt - n / p) <= (1 << dim) + 1e-9), (l, cnt, n)


# ------------------------------------------------------------------ two-level closed form
def _cheb_propagator(A, Dinv, lam, m):
    """E_m = p_m(D^-1 A), p_m(t) = T_m((theta - t)/delta) / T_m(theta/delta) over
    [0.08 lam, 1.2 lam], through the eigendecomposition of the
    symmetric D^-1/2 A D^-1/2 (SURVEY c.1 step 9: the first-kind Chebyshev
    error propagator)."""
    hi, lo = 1.2 * lam, 0.08 * lam
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    s = np.sqrt(Dinv)
    Bs = s[:, None] * A * s[None, :]
    w, V = np.linalg.eigh(Bs)
    Tm = npcheb.Chebyshev.basis(m)
    pm = Tm((theta - w) / delta) / Tm(theta / delta)
    return s[:, None] * ((V * pm) @ V.T) * (1.0 / s)[None, :]   # D^-1/2 p_m(Bs) D^1/2


def _two_level_closed_form(h, b):
    """The literal two-level cycle of P:318-327 with local smoothing,
    dense: level 1 split into S (smoothed) and E (refinement edge) rows."""
    l1, l0 = h.levels[1], h.levels[0]
    K1 = l1.K.toarray()
    S, E = l1.S, l1.E
    SE = S | E
    P = l1.P.toarray()
    m = h.degree
    A_SS = K1[np.ix_(S, S)]
    Em = _cheb_propagator(A_SS, l1.Dinv[S], l1.lam, m)
    G = (np.eye(int(S.sum())) - Em) @ np.linalg.inv(A_SS)
    # copy_to_mg: free leaf DoF n -> level lambda(n)
    d1 = np.zeros(l1.space.n)
    d0 = np.zeros(l0.space.n)
    for i in range(h.leaf.n_free):
        (d1 if h.leaf.lam[i] == 1 else d0)[h.lam_slot[i]] = b[i]
    assert np.all(d1[E] == 0)
    x1 = np.zeros(l1.space.n)
    x1[S] = G @ d1[S]                                  # pre-smoothing from 0
    r = np.where(SE, d1 - K1 @ x1, 0.0)                # residual with edge rows (E: -A^{ES} x^S)
    d0 = d0 + P.T @ r
    x0 = np.zeros(l0.space.n)
    if l0.S.any():
        A0 = l0.K.toarray()[np.ix_(l0.S, l0.S)]
        x0[l0.S] = np.linalg.solve(A0, d0[l0.S])      # coarse direct solve
    x1 = x1 + np.where(SE, P @ x0, 0.0)                # prolongation on S u E
    g = d1[S] - K1[np.ix_(S, E)] @ x1[E]               # post-smoother rhs d^S - A^{SE} x^E
    x1[S] = x1[S] + G @ (g - A_SS @ x1[S])             # post-smoothing
    u = np.empty(h.leaf.n_free)
    for i in range(h.leaf.n_free):
        u[i] = (x1 if h.leaf.lam[i] == 1 else x0)[h.lam_slot[i]]
    return u, G, A_SS, P, K1


def _brick2x2():
    return F.coarse_forest(2, [(0, 0), (1, 0), (0, 1), (1, 1)])


@pytest.mark.parametrize("k", [1, 2])
def test_two_level_uniform_is_textbook_two_grid(k):
    """Uniform two-level mesh (2x2 brick refined once): no edge rows, and the
    oracle's V-cycle equals the textbook two-grid cycle u3 = u2 + G (b - A u2),
    u2 = u1 + P A_0^-1 P^T (b - A u1), u1 = G b, G = (I - E_m) A^-1."""
    f = F.refine(_brick2x2(), np.ones(4, dtype=bool))
    h = mg.build(f, k)
    assert h.L == 1 and not h.levels[1].E.any()
    b = np.random.default_rng(11).uniform(-1, 1, h.leaf.n_free)
    u, G, A, P, K1 = _two_level_closed_form(h, b)
    # textbook form in the level-1 ordering (every free leaf DoF has lambda = 1)
    assert np.all(h.leaf.lam == 1)
    bb = np.zeros(h.levels[1].space.n)
    bb[h.lam_slot] = b
    S = h.levels[1].S
    l0 = h.levels[0]
    A0 = l0.K.toarray()[np.ix_(l0.S, l0.S)]
    PS = P[np.ix_(S, l0.S)]
    u1 = G @ bb[S]
    u2 = u1 + PS @ np.linalg.solve(A0, PS.T @ (bb[S] - A @ u1))
    u3 = u2 + G @ (bb[S] - A @ u2)
    assert np.abs(u3[h.lam_slot] - u).max() <= 1e-13 * np.abs(u).max()
    got = mg.vcycle(h, b)
    assert np.abs(got - u).max() <= 1e-12 * np.abs(u).max()


@pytest.mark.parametrize("k,tree", [(1, 0), (2, 0), (2, 3)])
def test_two_level_local_smoothing_closed_form(k, tree):
    """Adaptive two-level mesh (2x2 brick, one tree refined): level 1 has edge
    rows E on the interface to the level-0 leaves; the oracle's V-cycle equals
    the dense closed form with the edge terms of P:439-469."""
    f0 = _brick2x2()
    m = np.zeros(4, dtype=bool)
    m[tree] = True
    f = F.close(F.refine(f0, m))
    h = mg.build(f, k)
    assert h.L == 1 and h.levels[1].E.any() and (h.leaf.lam == 0).any()
    b = np.random.default_rng(12 + tree).uniform(-1, 1, h.leaf.n_free)
    u, *_ = _two_level_closed_form(h, b)
    got = mg.vcycle(h, b)
    assert np.abs(got - u).max() <= 1e-12 * np.abs(u).max(), np.abs(got - u).max()


def test_chebyshev_propagator_matches_recurrence_on_a_level():
    """The dense T_m propagator equals the oracle's recurrence from x0 = 0 on an
    adaptive level with E rows (x = (I - E_m) (A^S)^-1 g on S)."""
    f = F.close(F.refine(_brick2x2(), np.array([True, False, False, True])))
    f = F.close(F.refine(f, (np.arange(f.n_leaves) % 3) == 0))
    h = mg.build(f, 2)
    lev = h.levels[h.L]
    S = lev.S
    g = np.random.default_rng(5).uniform(-1, 1, lev.space.n) * S
    A_SS = lev.K.toarray()[np.ix_(S, S)]
    Em = _cheb_propagator(A_SS, lev.Dinv[S], lev.lam, h.degree)
    want = (np.eye(int(S.sum())) - Em) @ np.linalg.solve(A_SS, g[S])
    got = mg.chebyshev(lev, g, None, h.degree)
    assert np.abs(got[S] - want).max() <= 1e-12 * np.abs(want).max()
    assert np.all(got[~S] == 0)


# ------------------------------------------------------------------ adaptive SPD, Neumann kernel
def _adaptive(dim, k):
    f = F.coarse_forest(dim, [(0,) * dim])
    for _ in range(2 if dim == 2 else 1):
        f = F.refine(f, np.ones(f.n_leaves, dtype=bool))
    for step in range(2):
        f = F.close(F.refine(f, (np.arange(f.n_leaves) % (3 + step)) == 0))
    return f


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_adaptive_levels_spd(dim, k):
    f = _adaptive(dim, k)
    h = mg.build(f, k, eig=False)
    n_edge_levels = 0
    for lev in h.levels:
        K = lev.K.toarray()
        if K.size == 0:
            continue
        assert np.abs(K - K.T).max() <= 1e-15 * np.abs(K).max()
        if lev.S.any():
            A = K[np.ix_(lev.S, lev.S)]
            np.linalg.cholesky(A)
            assert np.linalg.eigvalsh(A).min() > 0
        n_edge_levels += int(lev.E.any())
    assert n_edge_levels >= 1


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_element_matrices_annihilate_constants(dim, k):
    for h in (1.0, 0.5, 0.125):
        Ae = fem.element_laplace(dim, k, h, 1.7)
        assert np.abs(Ae @ np.ones(Ae.shape[0])).max() <= 1e-13 * np.abs(Ae).max()
    # config-4 sub-box element matrices (levels 0-1 integrate a over level-2 sub-boxes)
    rng = np.random.default_rng(3)
    for nsub in (2, 4):
        coefs = 10.0 ** rng.uniform(-2, 2, nsub ** dim)
        Ae = fem.element_laplace_subbox(dim, k, 0.5, coefs, nsub)
        assert np.abs(Ae - Ae.T).max() <= 1e-13 * np.abs(Ae).max()
        assert np.abs(Ae @ np.ones(Ae.shape[0])).max() <= 1e-12 * np.abs(Ae).max()
        assert np.linalg.eigvalsh(Ae)[1] > 0            # kernel = constants only


@pytest.mark.parametrize("dim,k", [(2, 2), (3, 1)])
def test_adaptive_level_operator_is_dirichlet_restriction_of_neumann(dim, k):
    """Assemble every level's cell operator over ALL level nodes (boundary
    included): K_full 1 = 0 (Neumann kernel), and deleting the Dirichlet rows and
    columns gives exactly the oracle's K_l."""
    f = _adaptive(dim, k)
    h = mg.build(f, k, eig=False)
    lat = h.lat
    for lev in h.levels:
        s = lev.space
        X = lat.cell_nodes(s.level, s.cells.gc)               # [nc, nn, d]
        keys = lat.lin(X.reshape(-1, dim))
        uk, inv = np.unique(keys, return_inverse=True)
        cd = inv.reshape(X.shape[0], X.shape[1])
        elem = fem.cell_element_matrices(dim, k, s.level, s.cells.gc, None)
        Kf = fem.assemble_cells(cd, elem, uk.size).toarray()
        assert np.abs(Kf @ np.ones(uk.size)).max() <= 1e-13 * np.abs(Kf).max()
        if s.n == 0:
            continue
        pos = np.searchsorted(uk, lat.lin(s.X))               # free nodes inside the full numbering
        assert np.array_equal(uk[pos], lat.lin(s.X))
        assert np.abs(Kf[np.ix_(pos, pos)] - lev.K.toarray()).max() <= 1e-14 * np.abs(Kf).max()
