"""Local-smoothing multigrid V-cycle and GMG-preconditioned CG (oracle).
TEST INFRASTRUCTURE ONLY.

Level-cell storage of the paper's algorithm:

* V-cycle with local smoothing (only V_l^S is smoothed,
  x^I and x^L pass through), restriction structure (identity on
  V_l^L, so lower-level parts of the defect already live on the lower levels),
  and block residual with edge matrices (r^S, r^I from A^S, A^{SI},
  A^{IS}; A^{SL} = A^{LS} = 0; r^L deferred).  Per level l >= 1 (SURVEY c.1
  step 11):
      1. x = 0;  x^S = Cheb(A^S, d^S, 0)
      2. r = d - K_l x on S u E rows          (E rows: -A^{ES} x^S)
      3. d_{l-1} += P_l^T r
      4. V(l-1)
      5. x^{S u E} += (P_l x_{l-1})^{S u E}
      6. x^S = Cheb(A^S, d^S - A^{SE} x^E, x^S)
  and x_0^S = (A_0^S)^{-1} d_0^S at l = 0 (direct coarse solver P:331),
  or -- coarse="chebyshev", P:890-895 -- x_0^S = Chebyshev iteration from 0 on
  D^{-1} A_0^S over the full eigenvalue range [lambda_min, lambda_max] of the
  Lanczos tridiagonal of a Jacobi-PCG run to relative unpreconditioned residual
  1e-3, with the smallest degree m whose a priori bound
  2 rho^m / (1 + rho^(2m)) (rho = (sqrt(kappa) - 1)/(sqrt(kappa) + 1),
  kappa = lambda_max / lambda_min) is <= 1e-3 (reading R28).
  copy_to_mg: d_{lambda(n)}[n] = b[n]; copy_from_mg: u[n] = x_{lambda(n)}[n].
* Chebyshev-Jacobi smoother: first-kind Chebyshev iteration on
  D^{-1} A^S over [0.08 lambda, 1.2 lambda] (reading R7/R8), degree m = 4
  (reading R6), recurrence of SURVEY c.1 step 9.
* Eigenvalue estimate: CG (Jacobi preconditioned, reading R9) for
  min(10, n_S) iterations from x = 0 on the right-hand side
  (-5.5, -4.5, ..., 5.5, -5.5, ...) over the S DoFs in canonical order
  (reading R10), Lanczos tridiagonal from the CG coefficients, lambda = its
  largest eigenvalue.
* Outer CG: x_0 = 0, stop on ||b - A x|| <= rtol ||b||
  (unpreconditioned residual), preconditioned by one V-cycle.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import fem
from .spmv import mv
from .forest import Forest
from .partition import level_cells, leaf_owners, LevelCells
from .spaces import Lattice, LevelSpace, LeafSpace, level_space, leaf_space, leaf_level_sets, S_CLASS, E_CLASS


CHEB_LO, CHEB_HI = 0.08, 1.2


@dataclass
class Level:
    space: LevelSpace
    K: sp.csr_matrix           # K_l on D_l \ B_l
    S: np.ndarray              # bool mask
    E: np.ndarray              # bool mask
    Dinv: np.ndarray           # 1/diag(A^S) on S, 0 on E
    P: sp.csr_matrix | None    # fine l <- coarse l-1
    lam: float = 0.0


@dataclass
class Hierarchy:
    forest: Forest
    lat: Lattice
    cells: list
    levels: list
    leaf: LeafSpace
    A_leaf: sp.csr_matrix
    b_leaf: np.ndarray
    degree: int = 4
    coarse_factor: object = None
    coarse_cheb: object = None      # (lambda_min, lambda_max, degree) for coarse="chebyshev"
    lam_slot: list = field(default_factory=list)   # per level: (level index of free DoFs)

    @property
    def L(self) -> int:
        return len(self.levels) - 1


@dataclass
class Topology:
    """Integer view (no matrices): level spaces, leaf space, lambda slots and
    the global leaf numbering (owner = owner of the level-lambda(n) DoF,
    DESIGN.md reading R25; sorted by (owner, Morton key))."""
    lat: Lattice
    cells: list
    spaces: list
    leaf: LeafSpace
    leaf_owner: np.ndarray      # per free DoF (canonical free order)
    leaf_global: np.ndarray     # permutation: global position -> canonical free index


def topology(f: Forest, k: int, n_ranks: int = 1) -> Topology:
    lat = Lattice(f, k)
    owners = leaf_owners(f, n_ranks)
    cells = level_cells(f, owners)
    leafsets = leaf_level_sets(f, lat)
    spaces = [level_space(f, lat, c, leafsets, cells[l - 1] if l else None) for l, c in enumerate(cells)]
    leaf = leaf_space(f, lat, owners, spaces, lambda xi: fem.lagrange(k, xi))
    fX = leaf.X[leaf.free_index >= 0]
    own = np.empty(leaf.n_free, dtype=np.int64)
    for l, s in enumerate(spaces):
        sel = np.nonzero(leaf.lam == l)[0]
        if sel.size == 0:
            continue
        lk = lat.lin(s.X)
        o = np.argsort(lk)
        q = lat.lin(fX[sel])
        p = o[np.searchsorted(lk[o], q)]
        own[sel] = s.owner[p]
    fkey = leaf.key[leaf.free_index >= 0]
    glob = np.lexsort((fkey, own))
    return Topology(lat, cells, spaces, leaf, own, glob)


def build(f: Forest, k: int, n_ranks: int = 1, coef_level2: np.ndarray | None = None,
          degree: int = 4, eig=True, rhs="one", coarse: str = "cholesky") -> Hierarchy:
    lat = Lattice(f, k)
    owners = leaf_owners(f, n_ranks)
    cells = level_cells(f, owners)
    leafsets = leaf_level_sets(f, lat)
    spaces = [level_space(f, lat, c, leafsets, cells[l - 1] if l else None) for l, c in enumerate(cells)]
    coef = None
    if coef_level2 is not None:
        coef = fem.Coefficient(np.asarray(coef_level2, dtype=np.float64), cells[2].gc, lat.R)
    levels = []
    for l, s in enumerate(spaces):
        K = fem.level_matrix(s, lat, coef)
        S = s.cls == S_CLASS
        E = s.cls == E_CLASS
        diag = K.diagonal()
        Dinv = np.zeros(s.n)
        if np.any(diag[S] <= 0):
            raise ZeroDivisionError("zero diagonal on an S row")
        Dinv[S] = 1.0 / diag[S]
        P = fem.transfer_matrix(s, spaces[l - 1], lat) if l > 0 else None
        levels.append(Level(s, K, S, E, Dinv, P))
    leaf = leaf_space(f, lat, owners, spaces, lambda xi: fem.lagrange(k, xi))
    A_leaf, b_leaf = fem.leaf_system(f, leaf, lat, coef, rhs=rhs)
    h = Hierarchy(f, lat, cells, levels, leaf, A_leaf, b_leaf, degree)
    # lambda slots: index of each free leaf DoF in its level's canonical order
    fX = leaf.X[leaf.free_index >= 0]
    slots = np.empty(leaf.n_free, dtype=np.int64)
    for l, lev in enumerate(levels):
        sel = np.nonzero(leaf.lam == l)[0]
        if sel.size == 0:
            continue
        lk = lat.lin(lev.space.X)
        o = np.argsort(lk)
        q = lat.lin(fX[sel])
        p = o[np.searchsorted(lk[o], q)]
        assert np.all(lk[p] == q)
        slots[sel] = p
    h.lam_slot = slots
    # coarse solver: dense Cholesky of A_0^S or a priori Chebyshev
    l0 = levels[0]
    nS0 = int(l0.S.sum())
    if nS0 and coarse == "cholesky":
        A0 = l0.K[l0.S][:, l0.S].toarray()
        h.coarse_factor = sla.cho_factor(A0)
    elif nS0 and coarse == "chebyshev":
        h.coarse_cheb = coarse_chebyshev_setup(l0)
    elif coarse not in ("cholesky", "chebyshev"):
        raise ValueError(coarse)
    if eig:
        for l in range(1, len(levels)):
            levels[l].lam = eigen_estimate(levels[l])
    return h


# --------------------------------------------------------------------------
# eigenvalue estimate
# --------------------------------------------------------------------------

def eigen_rhs(lev: Level) -> np.ndarray:
    """(-5.5, -4.5, ..., 5.5, -5.5, ...) over the S DoFs in canonical order."""
    v = np.zeros(lev.space.n)
    sidx = np.nonzero(lev.S)[0]
    v[sidx] = -5.5 + (np.arange(sidx.size) % 12)
    return v


def cg_lanczos(A, Dinv, v, maxit, tol=1e-10):
    """Jacobi-PCG on A x = v from x = 0; returns (alphas, betas)."""
    r = v.copy()
    z = Dinv * r
    p = z.copy()
    rz = float(r @ z)
    r0 = float(np.linalg.norm(r))
    alphas, betas = [], []
    if rz == 0.0 or r0 == 0.0:
        return alphas, betas
    for it in range(maxit):
        q = A @ p
        pq = float(p @ q)
        alpha = rz / pq
        alphas.append(alpha)
        r = r - alpha * q
        if it == maxit - 1:
            break
        z = Dinv * r
        rz_new = float(r @ z)
        if np.linalg.norm(r) <= tol * r0 or rz_new == 0.0:
            break
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    return alphas, betas


def lanczos_tridiag(alphas, betas) -> np.ndarray:
    m = len(alphas)
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
        if j > 0:
            T[j, j - 1] = T[j - 1, j] = np.sqrt(betas[j - 1]) / alphas[j - 1]
    return T


def eigen_estimate(lev: Level, iters: int = 10) -> float:
    nS = int(lev.S.sum())
    if nS == 0:
        return 0.0
    S = lev.S
    A_S = lev.K[S][:, S]                  # A_l^S, the matrix of the smoother (R9)
    alphas, betas = cg_lanczos(A_S, lev.Dinv[S], eigen_rhs(lev)[S], min(iters, nS))
    if not alphas:
        return 0.0
    T = lanczos_tridiag(alphas, betas)
    return float(np.linalg.eigvalsh(T).max())


COARSE_REDUCTION = 1e-3      # P:892-893 "residual reduction by 10^3"
COARSE_CG_TOL = 1e-3         # P:894-895 "relative tolerance ... of 10^-3"


def chebyshev_degree(kappa: float, eps: float = COARSE_REDUCTION) -> int:
    """Smallest m with the classical Chebyshev bound 2 rho^m / (1 + rho^(2m)) <= eps,
    rho = (sqrt(kappa) - 1) / (sqrt(kappa) + 1)."""
    if kappa <= 1.0 + 1e-12:
        return 1
    rho = (np.sqrt(kappa) - 1.0) / (np.sqrt(kappa) + 1.0)
    m = 1
    while 2.0 * rho ** m / (1.0 + rho ** (2 * m)) > eps:
        m += 1
    return m


def coarse_chebyshev_setup(lev: Level):
    """(lambda_min, lambda_max, degree) of the coarse Chebyshev solver."""
    nS = int(lev.S.sum())
    S = lev.S
    alphas, betas = cg_lanczos(lev.K[S][:, S], lev.Dinv[S], eigen_rhs(lev)[S], nS, tol=COARSE_CG_TOL)
    ev = np.linalg.eigvalsh(lanczos_tridiag(alphas, betas))
    lo, hi = float(ev.min()), float(ev.max())
    return lo, hi, chebyshev_degree(hi / lo)


def chebyshev_range(lev: Level, g: np.ndarray, lam_lo: float, lam_hi: float, degree: int) -> np.ndarray:
    """First-kind Chebyshev-Jacobi from x = 0 over [lam_lo, lam_hi] (SURVEY c.1 step 9)."""
    theta = 0.5 * (lam_hi + lam_lo)
    delta = 0.5 * (lam_hi - lam_lo)
    A, Dinv = lev.K, lev.Dinv
    x = np.zeros_like(g)
    r = Dinv * g
    if delta <= 1e-14 * theta:              # one eigenvalue: the first step is exact
        return r / theta
    sigma = theta / delta
    rho = 1.0 / sigma
    dvec = r / theta
    for j in range(degree):
        x = x + dvec
        if j < degree - 1:
            r = r - Dinv * mv(A, dvec)
            rho_new = 1.0 / (2.0 * sigma - rho)
            dvec = rho_new * rho * dvec + (2.0 * rho_new / delta) * r
            rho = rho_new
    return x


# --------------------------------------------------------------------------
# smoother and V-cycle
# --------------------------------------------------------------------------

def chebyshev(lev: Level, g: np.ndarray, x0: np.ndarray | None, degree: int) -> np.ndarray:
    """First-kind Chebyshev-Jacobi on S rows (SURVEY c.1 step 9).  With x0 the
    initial residual includes the edge term: D^-1 (g - K x0) on S rows equals
    D^-1 (g^S - A^S x^S - A^{SE} x^E)."""
    lam_hi = CHEB_HI * lev.lam
    lam_lo = CHEB_LO * lev.lam
    theta = 0.5 * (lam_hi + lam_lo)
    delta = 0.5 * (lam_hi - lam_lo)
    sigma = theta / delta
    A, Dinv = lev.K, lev.Dinv
    if x0 is None:
        x = np.zeros_like(g)
        r = Dinv * g
    else:
        x = x0.copy()
        r = Dinv * (g - mv(A, x))
    rho = 1.0 / sigma
    dvec = r / theta
    for j in range(degree):
        x = x + dvec
        if j < degree - 1:
            r = r - Dinv * mv(A, dvec)
            rho_new = 1.0 / (2.0 * sigma - rho)
            dvec = rho_new * rho * dvec + (2.0 * rho_new / delta) * r
            rho = rho_new
    return x


def coarse_solve(h: Hierarchy, d0: np.ndarray) -> np.ndarray:
    lev = h.levels[0]
    x = np.zeros_like(d0)
    if h.coarse_factor is not None:
        x[lev.S] = sla.cho_solve(h.coarse_factor, d0[lev.S])
    elif getattr(h, "coarse_cheb", None) is not None:
        lo, hi, m = h.coarse_cheb
        x = chebyshev_range(lev, d0 * lev.S, lo, hi, m)
    return x


def vcycle_levels(h: Hierarchy, d: list) -> list:
    """V(L) on level defects d_l (modified in place: restriction adds to d_{l-1})."""
    L = h.L
    x = [None] * (L + 1)

    def V(l):
        lev = h.levels[l]
        if l == 0:
            x[0] = coarse_solve(h, d[0])
            return
        xl = chebyshev(lev, d[l], None, h.degree)                    # 1
        SE = lev.S | lev.E
        r = np.where(SE, d[l] - mv(lev.K, xl), 0.0)                  # 2
        d[l - 1] = d[l - 1] + lev.P.T @ r                            # 3
        V(l - 1)                                                     # 4
        xl = xl + np.where(SE, lev.P @ x[l - 1], 0.0)                # 5
        x[l] = chebyshev(lev, d[l], xl, h.degree)                    # 6

    V(L)
    return x


def copy_to_mg(h: Hierarchy, b: np.ndarray) -> list:
    d = [np.zeros(lev.space.n) for lev in h.levels]
    for l in range(h.L + 1):
        sel = h.leaf.lam == l
        d[l][h.lam_slot[sel]] = b[sel]
    return d


def copy_from_mg(h: Hierarchy, x: list) -> np.ndarray:
    u = np.zeros(h.leaf.n_free)
    for l in range(h.L + 1):
        sel = h.leaf.lam == l
        u[sel] = x[l][h.lam_slot[sel]]
    return u


def vcycle(h: Hierarchy, b: np.ndarray) -> np.ndarray:
    """One V-cycle preconditioner application on the free leaf DoFs."""
    return copy_from_mg(h, vcycle_levels(h, copy_to_mg(h, b)))


def pcg(h: Hierarchy, b: np.ndarray, rtol: float = 1e-8, maxit: int = 200, precond=None):
    """CG on the leaf system, x0 = 0, stop at the first k whose residual norm
    ||r_k|| <= rtol ||b|| (unpreconditioned 2-norm).  r_k is CG's
    recursively updated residual r_k = r_{k-1} - alpha A p, equal to b - A x_k in
    exact arithmetic; the tests check the true residual of the returned x
    separately."""
    A = h.A_leaf
    M = (lambda r: vcycle(h, r)) if precond is None else precond
    x = np.zeros_like(b)
    r = b.copy()
    nb = float(np.linalg.norm(b))
    hist = [1.0 if nb else 0.0]
    if nb == 0.0:
        return x, 0, 0.0, hist
    z = M(r)
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, maxit + 1):
        q = mv(A, p)
        alpha = rz / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        rel = float(np.linalg.norm(r)) / nb
        hist.append(rel)
        if rel <= rtol:
            return x, it, rel, hist
        z = M(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    return x, maxit, hist[-1], hist
