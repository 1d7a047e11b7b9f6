"""Level and leaf DoF spaces (oracle).  TEST INFRASTRUCTURE ONLY.

Definitions (§2.3; notation of SURVEY.md §0):

* M_l = C_l U {leaves of level < l}; C_l = cells of level exactly l.
* D_l = the Q_k nodes of the C_l cells ("level DoFs"), B_l = D_l on the
  boundary of Omega (homogeneous Dirichlet), E_l = nodes of D_l \\ B_l
  lying on the closure of a leaf of level < l (the fine-side representation of
  the refinement edge V_l^I), S_l = D_l \\ (E_l U B_l) -- the DoFs of
  V_l^S on which the local smoother acts.
* Leaf mesh M_L = the leaves; a leaf node is *hanging* when it lies
  on the closure of a leaf T without being a node of T ("elimination of
  hanging nodes"); its value is the Q_k interpolant of T.
* lambda(n) = max{ l : node n in S_l } for a free leaf DoF n (copy_to_mg /
  copy_from_mg of SURVEY §8(a) a9).

All nodes live on one integer lattice: local node a of cell (l, G) sits at
X = (k G + a) 2^(L - l), L the finest level.  The canonical order of a set of
nodes is the Morton order of X (x fastest, reading R10); the global
(rank-aware) order sorts by (owner, Morton).  Owner of a level-l node (DESIGN.md
reading R25; PAPER.md:519-521 leaves the interface rule open): level 0 -> rank
0 (coarse handoff); l >= 1 -> min over the level-l cells that have the node of
the owner of the cell's PARENT, i.e. of the rank that computes the cell's
family (first-child rule).  Pinned by hand-derived values and a
brute-force evaluation in tests/test_oracle_r2_pins.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .forest import Forest, morton, nbits_for
from .partition import LevelCells


def local_offsets(dim: int, k: int) -> np.ndarray:
    """Local node multi-indices a in [0,k]^d, x fastest: [(k+1)^d, d]."""
    n1 = k + 1
    idx = np.arange(n1 ** dim)
    return np.stack([(idx // n1 ** j) % n1 for j in range(dim)], axis=1).astype(np.int64)


class Lattice:
    """Finest node lattice of a forest for degree k."""

    def __init__(self, f: Forest, k: int):
        self.dim = f.dim
        self.k = k
        self.L = f.max_level
        self.trees = f.trees
        self.ext = f.brick_extent()
        self.T = k << self.L                         # tree edge in lattice units
        self.R = int(self.ext.max()) * self.T + 3    # radix for scalar keys
        self.nbits = nbits_for(int(self.ext.max()) * self.T + 1)
        occ = np.zeros(tuple(self.ext), dtype=bool)
        occ[tuple(self.trees.T)] = True
        self.occ = occ

    def lin(self, X: np.ndarray) -> np.ndarray:
        key = np.zeros(X.shape[0], dtype=np.int64)
        for j in range(self.dim - 1, -1, -1):
            key = key * self.R + (X[:, j] + 1)
        return key

    def unlin(self, key: np.ndarray) -> np.ndarray:
        X = np.empty((key.size, self.dim), dtype=np.int64)
        rem = key.copy()
        for j in range(self.dim):
            X[:, j] = rem % self.R - 1
            rem //= self.R
        return X

    def morton(self, X: np.ndarray) -> np.ndarray:
        return morton(X, self.nbits)

    def cell_nodes(self, level: int, gc: np.ndarray) -> np.ndarray:
        """[n_cells, (k+1)^d, d] lattice coordinates of the cells' nodes."""
        off = local_offsets(self.dim, self.k)
        return ((self.k * gc[:, None, :] + off[None, :, :]) << (self.L - level))

    def on_boundary(self, X: np.ndarray) -> np.ndarray:
        """x on the boundary of Omega <=> some point x + eps*s (s in {-1,1}^d)
        lies outside every tree of the brick."""
        out = np.zeros(X.shape[0], dtype=bool)
        for c in range(1 << self.dim):
            tp = np.empty_like(X)
            for j in range(self.dim):
                tp[:, j] = X[:, j] // self.T if (c >> j) & 1 else (X[:, j] - 1) // self.T
            inside = np.all((tp >= 0) & (tp < self.ext), axis=1)
            tpc = np.clip(tp, 0, self.ext - 1)
            inside &= self.occ[tuple(tpc.T)]
            out |= ~inside
        return out

    def cells_containing(self, X: np.ndarray, level: int) -> list[np.ndarray]:
        """The (up to 2^d) level-`level` cells whose closure contains X, as
        global cell coordinates, one array per sign pattern."""
        s = self.k << (self.L - level)               # cell edge in lattice units
        out = []
        for c in range(1 << self.dim):
            q = np.empty_like(X)
            for j in range(self.dim):
                q[:, j] = X[:, j] // s if (c >> j) & 1 else (X[:, j] - 1) // s
            out.append(q)
        return out


def _cell_lin(gc: np.ndarray, R: int) -> np.ndarray:
    key = np.zeros(gc.shape[0], dtype=np.int64)
    for j in range(gc.shape[1] - 1, -1, -1):
        key = key * R + (gc[:, j] + 1)
    return key


S_CLASS, E_CLASS = 0, 1


@dataclass
class LevelSpace:
    level: int
    cells: LevelCells
    X: np.ndarray          # [n, d] canonical (Morton) order, D_l \ B_l
    key: np.ndarray        # Morton keys (canonical order, increasing)
    cls: np.ndarray        # uint8: 0 = S, 1 = E
    owner: np.ndarray      # DoF owner
    cell_dofs: np.ndarray  # [n_cells, (k+1)^d] canonical index, -1 for B
    n_boundary: int

    @property
    def n(self) -> int:
        return self.X.shape[0]

    def global_order(self) -> np.ndarray:
        """Permutation: position in (owner, Morton) order -> canonical index."""
        return np.lexsort((self.key, self.owner))


def leaf_level_sets(f: Forest, lat: Lattice) -> dict[int, np.ndarray]:
    """Sorted scalar keys of the leaves at each level (cell lattice)."""
    Rc = lat.R
    return {int(l): np.sort(_cell_lin(f.gc[f.level == l], Rc)) for l in np.unique(f.level)}


def parent_owner(cells: LevelCells, parents: LevelCells) -> np.ndarray:
    """Owner of the parent of every cell (the rank that computes its family)."""
    R = int(max(cells.gc.max(initial=0), parents.gc.max(initial=0))) + 3
    pk = _cell_lin(parents.gc, R)
    ck = _cell_lin(cells.gc >> 1, R)
    o = np.argsort(pk)
    idx = o[np.searchsorted(pk[o], ck)]
    assert np.all(pk[idx] == ck)
    return parents.owner[idx]


def level_space(f: Forest, lat: Lattice, cells: LevelCells, leafsets=None,
                parents: LevelCells | None = None) -> LevelSpace:
    """DoF owner (R25): level 0 -> rank 0 (coarse handoff); level l >= 1
    -> min over the cells having the node of the owner of their parent (the rank
    that computes the family)."""
    l = cells.level
    if leafsets is None:
        leafsets = leaf_level_sets(f, lat)
    nodes = lat.cell_nodes(l, cells.gc)                  # [nc, nn, d]
    nc, nn, d = nodes.shape
    flat = nodes.reshape(-1, d)
    lk = lat.lin(flat)
    uk, inv = np.unique(lk, return_inverse=True)
    UX = lat.unlin(uk)
    bnd = lat.on_boundary(UX)
    # E: on the closure of a leaf of level < l
    onE = np.zeros(uk.size, dtype=bool)
    for lc in range(l):
        if lc not in leafsets:
            continue
        ls = leafsets[lc]
        for q in lat.cells_containing(UX, lc):
            ck = _cell_lin(q, lat.R)
            pos = np.searchsorted(ls, ck)
            pos = np.minimum(pos, ls.size - 1)
            onE |= ls[pos] == ck
    keep = ~bnd
    mk = lat.morton(UX[keep])
    order = np.argsort(mk, kind="stable")
    X = UX[keep][order]
    key = mk[order]
    cls = np.where(onE[keep][order], E_CLASS, S_CLASS).astype(np.uint8)
    # unique-node -> canonical index
    canon = -np.ones(uk.size, dtype=np.int64)
    kept_ids = np.nonzero(keep)[0][order]
    canon[kept_ids] = np.arange(kept_ids.size)
    cell_dofs = canon[inv].reshape(nc, nn)
    own_u = np.full(uk.size, np.iinfo(np.int64).max, dtype=np.int64)
    if l == 0 or parents is None:
        own_u[:] = 0
    else:
        np.minimum.at(own_u, inv, np.repeat(parent_owner(cells, parents), nn))
    owner = own_u[kept_ids]
    return LevelSpace(l, cells, X, key, cls, owner, cell_dofs, int(bnd.sum()))


@dataclass
class LeafSpace:
    X: np.ndarray          # [n_all, d] all leaf nodes, sorted by Morton key
    key: np.ndarray
    hanging: np.ndarray    # bool
    dirichlet: np.ndarray  # bool
    free_index: np.ndarray # canonical free index or -1
    n_free: int
    owner: np.ndarray      # per node (min owner of leaves having it as a node)
    cell_nodes: np.ndarray # [n_leaves, (k+1)^d] index into X
    C: object              # scipy CSR [n_all, n_free] constraint matrix
    lam: np.ndarray        # lambda(n) for free DoFs (canonical free order)


def leaf_space(f: Forest, lat: Lattice, leaf_owner: np.ndarray, levels: list[LevelSpace],
               basis_1d) -> LeafSpace:
    import scipy.sparse as sp
    d, k, L = lat.dim, lat.k, lat.L
    nn = (k + 1) ** d
    allX = []
    for l in np.unique(f.level):
        sel = np.nonzero(f.level == l)[0]
        allX.append((sel, lat.cell_nodes(int(l), f.gc[sel])))
    cell_nodes_X = np.empty((f.n_leaves, nn, d), dtype=np.int64)
    for sel, Xs in allX:
        cell_nodes_X[sel] = Xs
    lk = lat.lin(cell_nodes_X.reshape(-1, d))
    uk, inv = np.unique(lk, return_inverse=True)
    UX = lat.unlin(uk)
    mk = lat.morton(UX)
    order = np.argsort(mk, kind="stable")
    X = UX[order]
    key = mk[order]
    pos = np.empty_like(order)
    pos[order] = np.arange(order.size)
    cell_nodes = pos[inv].reshape(f.n_leaves, nn)
    n_all = X.shape[0]
    dirichlet = lat.on_boundary(X)
    # hanging: on the closure of a leaf T without being one of T's nodes
    leafsets = leaf_level_sets(f, lat)
    hang_level = -np.ones(n_all, dtype=np.int64)
    hang_cell = np.zeros((n_all, d), dtype=np.int64)
    for lc, ls in leafsets.items():
        step = 1 << (L - lc)                           # T's node spacing
        off_lattice = np.any(X % step != 0, axis=1)
        for q in lat.cells_containing(X, lc):
            ck = _cell_lin(q, lat.R)
            p = np.minimum(np.searchsorted(ls, ck), ls.size - 1)
            hit = (ls[p] == ck) & off_lattice
            newh = hit & (hang_level < 0)
            hang_level[newh] = lc
            hang_cell[newh] = q[newh]
    # a hanging node on the boundary of Omega (3D: midpoint of a face edge that
    # lies on the boundary) is a Dirichlet node: its value is 0 either way
    hanging = (hang_level >= 0) & ~dirichlet
    free = ~hanging & ~dirichlet
    free_index = -np.ones(n_all, dtype=np.int64)
    free_index[free] = np.arange(int(free.sum()))
    n_free = int(free.sum())
    # constraints: value at hanging X = interpolant of the coarse leaf T
    rows = [np.nonzero(free)[0]]
    cols = [free_index[free]]
    vals = [np.ones(n_free)]
    hid = np.nonzero(hanging)[0]
    if hid.size:
        off = local_offsets(d, k)
        lev = hang_level[hid]
        G = hang_cell[hid]
        for lc in np.unique(lev):
            s_ = lev == lc
            h_ids = hid[s_]
            Gc = G[s_]
            cell_size = k << (L - int(lc))
            xi = (X[h_ids] - Gc * cell_size) / cell_size          # in [0,1]^d
            w = np.ones((h_ids.size, off.shape[0]))
            for j in range(d):
                w *= basis_1d(xi[:, j])[:, off[:, j]]
            mX = (lat.cell_nodes(int(lc), Gc))                     # [nh, nn, d]
            mkeys = lat.lin(mX.reshape(-1, d))
            allkeys = lat.lin(X)
            o2 = np.argsort(allkeys)
            p2 = o2[np.searchsorted(allkeys[o2], mkeys)]
            assert np.all(allkeys[p2] == mkeys), "master node not a leaf node"
            p2 = p2.reshape(h_ids.size, -1)
            assert not np.any(hanging[p2] & (np.abs(w) > 1e-14)), "chained hanging node"
            m_free = free_index[p2]
            ok = (m_free >= 0) & (np.abs(w) > 0)
            rows.append(np.repeat(h_ids, off.shape[0])[ok.ravel()])
            cols.append(m_free[ok])
            vals.append(w[ok])
    C = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n_all, n_free))
    # owner of a node = min owner of leaves having it as a node
    own = np.full(n_all, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(own, cell_nodes.ravel(), np.repeat(leaf_owner, nn))
    # lambda(n) = max{ l : n in S_l }
    lam = -np.ones(n_free, dtype=np.int64)
    fk = lat.lin(X[free])
    for ls_ in levels:
        sk = lat.lin(ls_.X[ls_.cls == S_CLASS])
        sk.sort()
        if sk.size == 0:
            continue
        p = np.minimum(np.searchsorted(sk, fk), sk.size - 1)
        hit = sk[p] == fk
        lam[hit] = np.maximum(lam[hit], ls_.level)
    assert np.all(lam >= 0), "free leaf DoF with no smoothing level"
    return LeafSpace(X, key, hanging, dirichlet, free_index, n_free, own, cell_nodes, C, lam)
