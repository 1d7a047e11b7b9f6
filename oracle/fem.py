"""Q_k finite elements on axis-parallel cells, assembled as explicit CSR
matrices (oracle).  TEST INFRASTRUCTURE ONLY.

* Weak form a(u,v) = int a grad u . grad v, f(v) = int f v, V = H^1_0 (P:148-155,
  variable coefficient for config 4).
* Nodal Q_k basis on [0,1]^d from equidistant interpolation points (
  GLL = equidistant for k <= 2, reading R14), tensor products with x
  the fastest local index.
* 1-D matrices by Gauss-Legendre quadrature of the Lagrange polynomials
  (K[a,b] = int phi_a' phi_b', M[a,b] = int phi_a phi_b); the element matrix of a
  cell of width h is a_T h^(d-2) sum_i (x)_j (j == i ? K : M) (tensor-product
  structure of P:575-577).  Cells coarser than the coefficient patches
  (config 4, levels 0-1) integrate the piecewise-constant coefficient exactly
  over their sub-boxes (reading R15).
* Level matrices: K_l assembled over C_l on D_l \\ B_l (Dirichlet
  rows/columns absent); A_l^S = K_l[S,S]; edge matrices A^{SE} = K_l[S,E],
  A^{ES} = K_l[E,S].
* Transfer P_l: row of fine node i = values at x_i of the coarse
  nodal basis of a parent cell whose closure contains x_i (each row written once);
  R_l = P_l^T.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .spaces import LevelSpace, LeafSpace, Lattice, local_offsets
from .partition import LevelCells


def nodes_1d(k: int) -> np.ndarray:
    if k > 2:
        raise NotImplementedError("k <= 2 (GLL = equidistant) only")
    return np.arange(k + 1) / k


def lagrange(k: int, xi: np.ndarray) -> np.ndarray:
    """[n, k+1] values of the 1-D Lagrange basis at points xi."""
    z = nodes_1d(k)
    xi = np.asarray(xi, dtype=np.float64)
    out = np.ones((xi.size, k + 1))
    for a in range(k + 1):
        for b in range(k + 1):
            if b != a:
                out[:, a] *= (xi - z[b]) / (z[a] - z[b])
    return out


def lagrange_deriv(k: int, xi: np.ndarray) -> np.ndarray:
    z = nodes_1d(k)
    xi = np.asarray(xi, dtype=np.float64)
    out = np.zeros((xi.size, k + 1))
    for a in range(k + 1):
        for c in range(k + 1):
            if c == a:
                continue
            term = np.full(xi.size, 1.0 / (z[a] - z[c]))
            for b in range(k + 1):
                if b != a and b != c:
                    term *= (xi - z[b]) / (z[a] - z[b])
            out[:, a] += term
    return out


def matrices_1d(k: int, lo: float = 0.0, hi: float = 1.0):
    """K, M on the reference interval restricted to the sub-interval [lo, hi]."""
    xg, wg = np.polynomial.legendre.leggauss(k + 2)
    x = lo + (hi - lo) * (xg + 1) / 2
    w = wg * (hi - lo) / 2
    P = lagrange(k, x)
    D = lagrange_deriv(k, x)
    K = (D * w[:, None]).T @ D
    M = (P * w[:, None]).T @ P
    # the exact matrices are symmetric; remove the rounding asymmetry of the sum
    return 0.5 * (K + K.T), 0.5 * (M + M.T)


def mass_weights_1d(k: int) -> np.ndarray:
    xg, wg = np.polynomial.legendre.leggauss(k + 2)
    x = (xg + 1) / 2
    return (lagrange(k, x) * (wg / 2)[:, None]).sum(axis=0)


def _kron_list(mats):
    """Kronecker product on the x-fastest local numbering: pass [m_x, m_y, (m_z)];
    the first entry acts on the fastest local index."""
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(m, out)
    return out


def element_laplace(dim: int, k: int, h: float, coef: float = 1.0) -> np.ndarray:
    K, M = matrices_1d(k)
    A = np.zeros(((k + 1) ** dim,) * 2)
    for i in range(dim):
        A += _kron_list([K if j == i else M for j in range(dim)])
    return coef * h ** (dim - 2) * A


def element_laplace_subbox(dim: int, k: int, h: float, coefs: np.ndarray, nsub: int) -> np.ndarray:
    """Element matrix of a cell split into nsub^d equal sub-boxes with constant
    coefficients coefs[sx + nsub*(sy + nsub*sz)] (exact integration)."""
    subs = [matrices_1d(k, s / nsub, (s + 1) / nsub) for s in range(nsub)]
    A = np.zeros(((k + 1) ** dim,) * 2)
    for sidx in range(nsub ** dim):
        sv = [(sidx // nsub ** j) % nsub for j in range(dim)]
        for i in range(dim):
            A += coefs[sidx] * _kron_list([subs[sv[j]][0] if j == i else subs[sv[j]][1]
                                           for j in range(dim)])
    return h ** (dim - 2) * A


class Coefficient:
    """Piecewise-constant coefficient a per level-2 cell (config 4), else 1."""

    def __init__(self, values_level2: np.ndarray | None, level2_gc: np.ndarray | None, R: int):
        self.values = values_level2
        self.R = R
        if values_level2 is not None:
            self.key = _lin(level2_gc, R)
            self.order = np.argsort(self.key)

    def lookup2(self, gc2: np.ndarray) -> np.ndarray:
        k = _lin(gc2, self.R)
        p = self.order[np.searchsorted(self.key[self.order], k)]
        assert np.all(self.key[p] == k)
        return self.values[p]


def _lin(gc, R):
    key = np.zeros(gc.shape[0], dtype=np.int64)
    for j in range(gc.shape[1] - 1, -1, -1):
        key = key * R + (gc[:, j] + 1)
    return key


def cell_element_matrices(dim, k, level, gc, coef: Coefficient | None):
    """Per-cell element matrices [n, nn, nn] (or one shared matrix)."""
    h = 2.0 ** (-level)
    if coef is None or coef.values is None:
        return element_laplace(dim, k, h)[None]
    if level >= 2:
        a = coef.lookup2(gc >> (level - 2))
        return a[:, None, None] * element_laplace(dim, k, h)[None]
    nsub = 1 << (2 - level)
    out = []
    offs = local_offsets(dim, nsub - 1) if nsub > 1 else np.zeros((1, dim), dtype=np.int64)
    for g in gc:
        gc2 = g[None, :] * nsub + offs
        out.append(element_laplace_subbox(dim, k, h, coef.lookup2(gc2), nsub))
    return np.stack(out)


def assemble_cells(cell_dofs: np.ndarray, elem: np.ndarray, n: int, cell_sel=None):
    """sum over cells of the element matrices scattered to cell_dofs (-1 dropped)."""
    cd = cell_dofs if cell_sel is None else cell_dofs[cell_sel]
    nc, nn = cd.shape
    if elem.shape[0] == 1:
        vals = np.broadcast_to(elem, (nc, nn, nn))
    else:
        vals = elem if cell_sel is None else elem[cell_sel]
    r = np.broadcast_to(cd[:, :, None], (nc, nn, nn)).ravel()
    c = np.broadcast_to(cd[:, None, :], (nc, nn, nn)).ravel()
    v = np.asarray(vals).ravel()
    ok = (r >= 0) & (c >= 0)
    return sp.csr_matrix((v[ok], (r[ok], c[ok])), shape=(n, n))


def level_matrix(ls: LevelSpace, lat: Lattice, coef: Coefficient | None):
    """K_l over all C_l cells (rows/cols D_l \\ B_l, canonical order)."""
    elem = cell_element_matrices(lat.dim, lat.k, ls.level, ls.cells.gc, coef)
    return assemble_cells(ls.cell_dofs, elem, ls.n)


def transfer_matrix(fine: LevelSpace, coarse: LevelSpace, lat: Lattice):
    """P_l: coarse (l-1) -> fine (l), CSR [n_fine, n_coarse]."""
    d, k = lat.dim, lat.k
    off = local_offsets(d, k)
    nn = off.shape[0]
    cells = fine.cells
    par_gc = cells.gc >> 1
    bits = cells.gc & 1
    # parent index in coarse cell list
    pk = _lin(par_gc, lat.R)
    ck = _lin(coarse.cells.gc, lat.R)
    o = np.argsort(ck)
    pidx = o[np.searchsorted(ck[o], pk)]
    assert np.all(ck[pidx] == pk)
    # first occurrence of each fine node (row written once)
    fd = fine.cell_dofs.ravel()
    first = np.full(fine.n, -1, dtype=np.int64)
    valid = np.nonzero(fd >= 0)[0]
    # reverse so that the earliest (cell, a) wins
    first[fd[valid[::-1]]] = valid[::-1]
    rows, cols, vals = [], [], []
    sel = first[first >= 0]
    cidx = sel // nn
    aidx = sel % nn
    xi = (bits[cidx] * k + off[aidx]) / (2.0 * k)         # [m, d] in parent coords
    w = np.ones((sel.size, nn))
    for j in range(d):
        w *= lagrange(k, xi[:, j])[:, off[:, j]]
    cdofs = coarse.cell_dofs[pidx[cidx]]                  # [m, nn]
    frow = fd[sel]
    ok = (cdofs >= 0) & (np.abs(w) > 0)
    rows = np.repeat(frow, nn)[ok.ravel()]
    cols = cdofs[ok]
    vals = w[ok]
    return sp.csr_matrix((vals, (rows, cols)), shape=(fine.n, coarse.n))


def leaf_system(f, leaf: LeafSpace, lat: Lattice, coef: Coefficient | None, rhs="one"):
    """A = C^T K_full C and b = C^T b_full on the free leaf DoFs (hanging nodes
    condensed into their masters, Dirichlet DoFs removed)."""
    d, k = lat.dim, lat.k
    nn = (k + 1) ** d
    n_all = leaf.X.shape[0]
    blocks = []
    bfull = np.zeros(n_all)
    mw = mass_weights_1d(k)
    mvec = _kron_list([mw[:, None] for _ in range(d)]).ravel()
    for l in np.unique(f.level):
        sel = np.nonzero(f.level == l)[0]
        elem = cell_element_matrices(d, k, int(l), f.gc[sel], coef)
        Kl = assemble_cells(leaf.cell_nodes[sel], elem, n_all)
        blocks.append(Kl)
        h = 2.0 ** (-int(l))
        if rhs == "one":
            np.add.at(bfull, leaf.cell_nodes[sel].ravel(), np.tile(mvec * h ** d, sel.size))
        elif callable(rhs):
            bl = _load_quadrature(d, k, int(l), f.gc[sel], rhs)
            np.add.at(bfull, leaf.cell_nodes[sel].ravel(), bl.ravel())
    Kfull = blocks[0]
    for b in blocks[1:]:
        Kfull = Kfull + b
    C = leaf.C
    A = (C.T @ Kfull @ C).tocsr()
    b = C.T @ bfull
    return A, b


def _load_quadrature(d, k, level, gc, f):
    nq = k + 3
    xg, wg = np.polynomial.legendre.leggauss(nq)
    x1 = (xg + 1) / 2
    w1 = wg / 2
    phi = lagrange(k, x1)                     # [nq, k+1]
    h = 2.0 ** (-level)
    off = local_offsets(d, k)
    qoff = local_offsets(d, nq - 1)
    out = np.zeros((gc.shape[0], off.shape[0]))
    for qi in range(qoff.shape[0]):
        q = qoff[qi]
        pts = (gc + x1[q][None, :]) * h
        fv = f(pts)
        w = np.prod(w1[q]) * h ** d
        ph = np.ones(off.shape[0])
        for j in range(d):
            ph = ph * phi[q[j], off[:, j]]
        out += (w * fv)[:, None] * ph[None, :]
    return out


def interpolate_leaf(leaf: LeafSpace, lat: Lattice, u) -> np.ndarray:
    """Nodal interpolant of a function on the free leaf DoFs."""
    X = leaf.X[leaf.free_index >= 0] / float(lat.T)
    return u(X)


def l2_error(f, leaf: LeafSpace, lat: Lattice, uh_free: np.ndarray, u) -> float:
    """|| u_h - u ||_{L2} with Gauss quadrature per leaf cell."""
    d, k = lat.dim, lat.k
    nq = k + 3
    xg, wg = np.polynomial.legendre.leggauss(nq)
    x1 = (xg + 1) / 2
    w1 = wg / 2
    phi = lagrange(k, x1)
    off = local_offsets(d, k)
    qoff = local_offsets(d, nq - 1)
    uall = leaf.C @ uh_free
    err = 0.0
    for l in np.unique(f.level):
        sel = np.nonzero(f.level == l)[0]
        h = 2.0 ** (-int(l))
        uc = uall[leaf.cell_nodes[sel]]
        for qi in range(qoff.shape[0]):
            q = qoff[qi]
            ph = np.ones(off.shape[0])
            for j in range(d):
                ph = ph * phi[q[j], off[:, j]]
            uhq = uc @ ph
            pts = (f.gc[sel] + x1[q][None, :]) * h
            e = uhq - u(pts)
            err += float(np.sum(np.prod(w1[q]) * h ** d * e * e))
    return float(np.sqrt(err))
