"""Dense "abstract" local-smoothing V-cycle (oracle checker).  TEST
INFRASTRUCTURE ONLY -- tiny forests (a few thousand nodes at most).

An independent, literal implementation of PAPER.md §2.2-2.3 used to pin the
level-cell-storage V-cycle of ``oracle.mg``:

* V_l is the conforming Q_k space on the level mesh M_l = C_l U {leaves of
  level < l} with the nodal basis, hanging nodes eliminated
   and homogeneous Dirichlet nodes removed.  Built generically
  from point evaluations: a hanging node's value is the interpolant of a cell
  on whose closure it lies without being one of its nodes (resolved
  recursively).
* A_l = restriction of a(.,.) to V_l; the embedding
  P: V_{l-1} -> V_l evaluates the coarse function at the fine nodes;
  R = P^T (Euclidean coefficient inner product).
* V_l = V^S + V^I + V^L by the support of each basis function: inside cells of
  level l (S), inside cells of level < l (L), straddling (I).
* Vcycle with the block smoother: only x^S is smoothed,
  by the Chebyshev-Jacobi method written as its error propagator
  E = T_m((theta - D^-1 A)/delta) / T_m(theta/delta) on the S block, computed by
  dense eigendecomposition (not the three-term recurrence of oracle.mg).
"""
from __future__ import annotations

import numpy as np


def _lagr(k, t):
    z = np.arange(k + 1) / k
    out = np.ones(k + 1)
    for a in range(k + 1):
        for b in range(k + 1):
            if b != a:
                out[a] *= (t - z[b]) / (z[a] - z[b])
    return out


def _K1M1(k):
    # exact 1-D matrices by high-order Gauss quadrature of the Lagrange basis
    xg, wg = np.polynomial.legendre.leggauss(8)
    x = (xg + 1) / 2
    w = wg / 2
    z = np.arange(k + 1) / k
    P = np.array([_lagr(k, t) for t in x])
    D = np.zeros_like(P)
    for a in range(k + 1):
        coeffs = np.poly1d([1.0])
        for b in range(k + 1):
            if b != a:
                coeffs = coeffs * np.poly1d([1.0, -z[b]]) / (z[a] - z[b])
        D[:, a] = np.polyder(coeffs)(x)
    K = (D * w[:, None]).T @ D
    M = (P * w[:, None]).T @ P
    return K, M


class Space:
    """Conforming Q_k space on a list of cells (level, G) of a brick forest."""

    def __init__(self, cells, dim, k, L, ext, occ):
        self.cells = cells
        self.dim, self.k, self.L = dim, k, L
        self.ext, self.occ = ext, occ
        nodes = {}
        self.cell_nodes = []
        for (l, G) in cells:
            s = 1 << (L - l)
            ids = []
            for a in np.ndindex(*([k + 1] * dim)):
                a = a[::-1]  # x fastest
                X = tuple((k * G[j] + a[j]) * s for j in range(dim))
                if X not in nodes:
                    nodes[X] = len(nodes)
                ids.append(nodes[X])
            self.cell_nodes.append(ids)
        self.X = list(nodes.keys())
        self.nid = nodes
        n = len(self.X)
        # containing cells of each node (closure)
        Xa = np.array(self.X, dtype=np.int64).reshape(n, dim)
        self.containing = [[] for _ in range(n)]
        for ci, (l, G) in enumerate(cells):
            cs = k << (L - l)
            lo = np.array(G, dtype=np.int64) * cs
            inside = np.all((Xa >= lo) & (Xa <= lo + cs), axis=1)
            for i in np.nonzero(inside)[0]:
                self.containing[i].append(ci)
        # hanging: in the closure of a cell without being one of its nodes
        self.hang_cell = [-1] * n
        for i, X in enumerate(self.X):
            for ci in self.containing[i]:
                l = cells[ci][0]
                if any(X[j] % (1 << (L - l)) for j in range(dim)):
                    if self.hang_cell[i] < 0 or cells[ci][0] < cells[self.hang_cell[i]][0]:
                        self.hang_cell[i] = ci
        self.boundary = [self._on_boundary(X) for X in self.X]
        self.free = [i for i in range(n) if self.hang_cell[i] < 0 and not self.boundary[i]]
        fpos = {i: q for q, i in enumerate(self.free)}
        # constraint matrix C: node values = C @ free coefficients
        C = np.zeros((n, len(self.free)))
        done = [False] * n

        def resolve(i):
            if done[i]:
                return
            if self.boundary[i]:
                pass
            elif self.hang_cell[i] < 0:
                C[i, fpos[i]] = 1.0
            else:
                ci = self.hang_cell[i]
                w = self.eval_weights(ci, self.X[i])
                for a, nj in enumerate(self.cell_nodes[ci]):
                    if w[a] != 0.0:
                        resolve(nj)
                        C[i] += w[a] * C[nj]
            done[i] = True

        for i in range(n):
            resolve(i)
        self.C = C

    def _on_boundary(self, X):
        T = self.k << self.L
        for c in range(1 << self.dim):
            tp = []
            for j in range(self.dim):
                tp.append(X[j] // T if (c >> j) & 1 else (X[j] - 1) // T)
            if any(t < 0 or t >= self.ext[j] for j, t in enumerate(tp)) or not self.occ[tuple(tp)]:
                return True
        return False

    def eval_weights(self, ci, X):
        l, G = self.cells[ci]
        cs = self.k << (self.L - l)
        w = np.ones(1)
        for j in range(self.dim):
            t = (X[j] - G[j] * cs) / cs
            w = np.kron(_lagr(self.k, t), w)
        return w

    def find_cell(self, X):
        k, L = self.k, self.L
        for ci, (l, G) in enumerate(self.cells):
            cs = k << (L - l)
            if all(G[j] * cs <= X[j] <= (G[j] + 1) * cs for j in range(self.dim)):
                return ci
        raise KeyError(X)

    def stiffness(self, coef_fn=None):
        K1, M1 = _K1M1(self.k)
        n = len(self.X)
        Kf = np.zeros((n, n))
        for ci, (l, G) in enumerate(self.cells):
            h = 2.0 ** (-l)
            Ae = np.zeros(((self.k + 1) ** self.dim,) * 2)
            for i in range(self.dim):
                m = np.ones((1, 1))
                for j in range(self.dim):
                    m = np.kron(K1 if j == i else M1, m)
                Ae += m
            Ae *= h ** (self.dim - 2) * (1.0 if coef_fn is None else coef_fn(l, G))
            ids = self.cell_nodes[ci]
            Kf[np.ix_(ids, ids)] += Ae
        return self.C.T @ Kf @ self.C

    def classify(self, level):
        """S / I / L of each free basis function by its support."""
        n = len(self.X)
        inc = np.zeros((len(self.cells), n))
        for ci, ids in enumerate(self.cell_nodes):
            inc[ci, ids] = 1.0
        sup = (inc @ (self.C != 0).astype(np.float64)) > 0      # [cells, free]
        lv = np.array([c[0] for c in self.cells])
        on_l = (sup & (lv == level)[:, None]).any(axis=0)
        below = (sup & (lv < level)[:, None]).any(axis=0)
        return np.where(on_l & ~below, "S", np.where(below & ~on_l, "L", "I"))


def embedding(coarse: Space, fine: Space) -> np.ndarray:
    """P: V_coarse -> V_fine, evaluation of the coarse function at fine nodes."""
    P = np.zeros((len(fine.free), len(coarse.free)))
    for q, i in enumerate(fine.free):
        X = fine.X[i]
        ci = coarse.find_cell(X)
        w = coarse.eval_weights(ci, X)
        for a, nj in enumerate(coarse.cell_nodes[ci]):
            P[q] += w[a] * coarse.C[nj]
    return P


def cheb_T(m, x):
    x = np.asarray(x, dtype=np.float64)
    return np.polynomial.chebyshev.chebval(x, [0] * m + [1])


def cheb_smooth_dense(A_S, g_S, x0_S, lam, m, lo=0.08, hi=1.2):
    """x = x0 + (I - E) A^-1 (g - A x0) with E = T_m((theta - D^-1 A)/delta)/T_m(theta/delta)."""
    Dg = np.diag(A_S).copy()
    Dh = 1.0 / np.sqrt(Dg)
    B = Dh[:, None] * A_S * Dh[None, :]
    mu, V = np.linalg.eigh(B)
    theta = 0.5 * (hi + lo) * lam
    delta = 0.5 * (hi - lo) * lam
    pm = (1.0 - cheb_T(m, (theta - mu) / delta) / cheb_T(m, theta / delta)) / mu
    r0 = g_S - A_S @ x0_S
    return x0_S + Dh * (V @ (pm * (V.T @ (Dh * r0))))


class AbstractMG:
    def __init__(self, forest, k, lams, degree=4, coef_fn=None):
        f = forest
        L = f.max_level
        self.L = L
        ext = f.brick_extent()
        occ = np.zeros(tuple(ext), dtype=bool)
        occ[tuple(f.trees.T)] = True
        # all cells of the forest by level
        allcells = set()
        for l, G in zip(f.level, f.gc):
            for m in range(int(l) + 1):
                allcells.add((m, tuple(int(v) for v in (G >> (int(l) - m)))))
        leaves = set((int(l), tuple(int(v) for v in G)) for l, G in zip(f.level, f.gc))
        self.spaces, self.A, self.cls = [], [], []
        for l in range(L + 1):
            cells = sorted([c for c in allcells if c[0] == l]) + \
                sorted([c for c in leaves if c[0] < l])
            sp = Space(cells, f.dim, k, L, ext, occ)
            self.spaces.append(sp)
            self.A.append(sp.stiffness(coef_fn))
            self.cls.append(sp.classify(l))
        self.P = [None] + [embedding(self.spaces[l - 1], self.spaces[l]) for l in range(1, L + 1)]
        self.lams = lams
        self.m = degree

    def smooth(self, l, u, g):
        S = self.cls[l] == "S"
        if not S.any():
            return u
        A = self.A[l]
        # g^S - A^{SI} x^I - A^{SL} x^L, initial x^S
        rhs = g[S] - A[np.ix_(S, ~S)] @ u[~S]
        out = u.copy()
        out[S] = cheb_smooth_dense(A[np.ix_(S, S)], rhs, u[S], self.lams[l], self.m)
        return out

    def vcycle(self, l, g):
        if l == 0:
            A0 = self.A[0]
            return np.linalg.solve(A0, g) if A0.size else np.zeros(0)
        u1 = self.smooth(l, np.zeros_like(g), g)
        r = g - self.A[l] @ u1
        u2 = u1 + self.P[l] @ self.vcycle(l - 1, self.P[l].T @ r)
        return self.smooth(l, u2, g)

    def leaf_keys(self):
        """Finest-lattice coordinates of the free leaf DoFs (level-L space)."""
        sp = self.spaces[self.L]
        return [sp.X[i] for i in sp.free]
