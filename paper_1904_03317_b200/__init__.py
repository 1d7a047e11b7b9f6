"""Thin Python binding of libgmg (include/gmg.h): argument marshalling only.

Every step of the hot path runs in the CUDA library ``libgmg.so`` built for
sm_100a from ``csrc/``; there is no Python or CPU fallback.  Importing this
package raises if the library has not been built (``__graft_entry__.build()``).
PyTorch is used only for device memory and streams (tensors are passed by
``data_ptr()``, the current torch stream is the launch stream).

Function names follow the C ABI (``gmg_forest_generate``, ``gmg_partition``,
``gmg_setup``, ``gmg_vcycle``, ``gmg_solve_cg`` ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GMG_LIB_PATH: an alternative build of the same library (A/B experiments with
# compile-time kernel variants); default the in-tree build
LIB_PATH = os.environ.get("GMG_LIB_PATH") or os.path.join(_HERE, "libgmg.so")

if "GMG_NCCL_LIB" not in os.environ:
    # use the libnccl that torch loads (pip nvidia-nccl), not the system copy
    try:
        import nvidia.nccl as _nccl_pkg
        for _p in _nccl_pkg.__path__:
            _cand = os.path.join(_p, "lib", "libnccl.so.2")
            if os.path.exists(_cand):
                os.environ["GMG_NCCL_LIB"] = _cand
                break
    except Exception:
        pass

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libgmg.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = C.CDLL(LIB_PATH)

# ------------------------------------------------------------------ status
GMG_OK = 0
STATUS = {0: "GMG_OK", 1: "GMG_E_INVALID_ARG", 2: "GMG_E_UNSORTED", 3: "GMG_E_NOT_TILING",
          4: "GMG_E_UNBALANCED", 5: "GMG_E_DEPTH", 6: "GMG_E_STATE", 7: "GMG_E_ZERO_DIAG",
          8: "GMG_E_SINGULAR_COARSE", 9: "GMG_E_NOT_CONVERGED", 10: "GMG_E_CUDA", 11: "GMG_E_NCCL",
          12: "GMG_E_OOM"}
GMG_CLOSE_BALANCE = 1
GMG_HOST_ONLY = 1
GMG_NO_GRAPH = 2
GMG_MIXED_PRECISION = 8
GMG_LOCAL_RANKS = 4
GMG_HOST_RANKS = 16
GMG_RANK_LOCAL = 32
GMG_EIG_KEY = 64
MAX_LEVELS = 64


class GmgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def _check(code):
    if code != GMG_OK:
        raise GmgError(code, _lib.gmg_last_error().decode())
    return code


# ------------------------------------------------------------------ structs
class Recipe(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_trees", C.c_int), ("tree_xyz", C.c_int32 * 24),
                ("global_refinements", C.c_int), ("rule", C.c_int), ("n_passes", C.c_int),
                ("center_num", C.c_int64 * 3), ("center_den", C.c_int64 * 3),
                ("radius_num", C.c_int64), ("radius_den", C.c_int64),
                ("shell_num", C.c_int64), ("shell_den", C.c_int64),
                ("corner", C.c_int64 * 3), ("s", C.c_int), ("lmax", C.c_int)]


class Model(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("n_ranks", C.c_int), ("W_opt_num", C.c_int64), ("W_opt_den", C.c_int64),
                ("W_sync", C.c_int64), ("W", C.c_int64), ("eta_num", C.c_int64), ("eta_den", C.c_int64),
                ("N", C.c_int64 * MAX_LEVELS), ("W_l", C.c_int64 * MAX_LEVELS),
                ("ghost_children", C.c_int64 * MAX_LEVELS), ("children", C.c_int64 * MAX_LEVELS)]


DEV_ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
DEV_FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class Params(C.Structure):
    _fields_ = [("k", C.c_int), ("cheb_degree", C.c_int), ("cheb_lo", C.c_double), ("cheb_hi", C.c_double),
                ("eig_iters", C.c_int), ("coef_level2", C.POINTER(C.c_double)), ("rank", C.c_int),
                ("n_ranks", C.c_int), ("nccl_comm", C.c_void_p), ("device", C.c_int), ("flags", C.c_uint32),
                ("coarse_solver", C.c_int), ("dev_alloc", DEV_ALLOC), ("dev_free", DEV_FREE),
                ("alloc_ctx", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [("dim", C.c_int), ("k", C.c_int), ("n_levels", C.c_int), ("n_ranks", C.c_int), ("rank", C.c_int),
                ("n_leaf_nodes", C.c_int64), ("n_leaf_free", C.c_int64), ("n_leaf_hanging", C.c_int64),
                ("n_leaf_dirichlet", C.c_int64), ("n_owned", C.c_int64), ("first_owned", C.c_int64),
                ("level_dofs", C.c_int64 * MAX_LEVELS), ("level_cells", C.c_int64 * MAX_LEVELS),
                ("level_families", C.c_int64 * MAX_LEVELS), ("level_S", C.c_int64 * MAX_LEVELS),
                ("level_E", C.c_int64 * MAX_LEVELS), ("level_B", C.c_int64 * MAX_LEVELS),
                ("level_leaf_cells", C.c_int64 * MAX_LEVELS), ("mg_vector_len", C.c_int64),
                ("level_r1", C.c_int64 * MAX_LEVELS), ("level_gf", C.c_int64 * MAX_LEVELS),
                ("small_levels", C.c_int64)]


class KernelStat(C.Structure):
    _fields_ = [("kind", C.c_int), ("level", C.c_int), ("launches", C.c_int64), ("seconds", C.c_double),
                ("bytes", C.c_double), ("bytes_layout", C.c_double)]


KERNEL_KINDS = ["apply", "cheb_x1", "cheb_11", "cheb_10", "cheb_01", "cheb_00", "cheb_p01", "cheb_stream",
                "cheb_stream_full", "restrict", "prolongate", "coarse", "exchange", "copy_mg", "leaf_apply", "other",
                "small_levels", "res_restrict"]

_vp = C.c_void_p
_i64p = C.POINTER(C.c_int64)
_SIGS = {
    "gmg_last_error": ([], C.c_char_p),
    "gmg_abi_version": ([], C.c_int),
    "gmg_forest_create": ([C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp, _vp, C.c_uint32, C.POINTER(_vp)], C.c_int),
    "gmg_forest_generate": ([C.POINTER(Recipe), C.POINTER(_vp)], C.c_int),
    "gmg_forest_sequence": ([C.c_int, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "gmg_forest_destroy": ([_vp], C.c_int),
    "gmg_forest_info": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), _i64p, C.POINTER(C.c_int)], C.c_int),
    "gmg_export_leaves": ([_vp, _vp, _vp, _vp], C.c_int),
    "gmg_partition": ([_vp, C.c_int, C.POINTER(_vp)], C.c_int),
    "gmg_partition_mode": ([_vp, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "gmg_partition_destroy": ([_vp], C.c_int),
    "gmg_partition_ex": ([_vp, C.c_int, C.c_int, C.c_int64, C.POINTER(_vp)], C.c_int),
    "gmg_partition_model": ([_vp, C.c_int64, C.POINTER(Model)], C.c_int),
    "gmg_export_tallies": ([_vp, _vp], C.c_int),
    "gmg_export_level_cells": ([_vp, C.c_int, _i64p, _vp, _vp, _vp], C.c_int),
    "gmg_params_default": ([C.POINTER(Params)], None),
    "gmg_setup": ([_vp, _vp, C.POINTER(Params), C.POINTER(_vp)], C.c_int),
    "gmg_hierarchy_destroy": ([_vp], C.c_int),
    "gmg_hierarchy_info": ([_vp, C.POINTER(Info)], C.c_int),
    "gmg_export_level_dofs": ([_vp, C.c_int, _i64p, _vp, _vp, _vp, _vp], C.c_int),
    "gmg_export_leaf_dofs": ([_vp, _i64p, _vp, _vp, _vp, _vp], C.c_int),
    "gmg_export_cell_dofs": ([_vp, C.c_int, _i64p, _vp], C.c_int),
    "gmg_vcycle": ([_vp, _vp, _vp, _vp], C.c_int),
    "gmg_solve_cg": ([_vp, _vp, _vp, C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double), _vp],
                     C.c_int),
    "gmg_rhs_constant": ([_vp, C.c_double, _vp, _vp], C.c_int),
    "gmg_level_apply": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "gmg_level_apply_kernel": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "gmg_level_apply_kernel_f32": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "gmg_get_coarse_chebyshev": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)], C.c_int),
    "gmg_restrict": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "gmg_prolongate": ([_vp, C.c_int, _vp, _vp, _vp], C.c_int),
    "gmg_leaf_apply": ([_vp, _vp, _vp, _vp], C.c_int),
    "gmg_level_smooth": ([_vp, C.c_int, _vp, _vp, C.c_int, _vp], C.c_int),
    "gmg_level_diagonal": ([_vp, C.c_int, _vp, _vp], C.c_int),
    "gmg_get_eigen": ([_vp, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "gmg_set_eigen": ([_vp, C.c_int, C.c_double], C.c_int),
    "gmg_launch_count": ([_vp, _i64p], C.c_int),
    "gmg_launch_profile": ([_vp, _i64p, _i64p], C.c_int),
    "gmg_export_rank_level": ([_vp, C.c_int, _i64p, _i64p, _i64p, _vp], C.c_int),
    "gmg_nccl_get_unique_id": ([C.c_char_p], C.c_int),
    "gmg_nccl_comm_init": ([C.c_char_p, C.c_int, C.c_int, C.POINTER(_vp)], C.c_int),
    "gmg_nccl_comm_destroy": ([_vp], C.c_int),
    "gmg_local_world_create": ([C.c_int, C.POINTER(_vp)], C.c_int),
    "gmg_local_world_destroy": ([_vp], C.c_int),
    "gmg_host_world_create": ([C.c_char_p, C.c_int, C.c_int, C.c_size_t, C.POINTER(_vp)], C.c_int),
    "gmg_host_world_destroy": ([_vp], C.c_int),
    "gmg_leaf_layout": ([_vp, _i64p, _i64p, _i64p], C.c_int),
    "gmg_forest_count_nodes": ([_vp, C.c_int, _i64p], C.c_int),
    "gmg_export_local_level": ([_vp, C.c_int, _i64p, _i64p, _vp, _vp, _vp, C.POINTER(C.c_int32), _vp, _vp, _vp,
                                _vp, _vp], C.c_int),
    "gmg_export_local_tables": ([_vp, C.c_int, _i64p, _i64p, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "gmg_export_owned_leaf_keys": ([_vp, _i64p, _vp, _vp], C.c_int),
    "gmg_profile_vcycle": ([_vp, _vp, _vp, C.c_int, C.POINTER(KernelStat), C.c_int, C.POINTER(C.c_int), _vp],
                           C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = sorted(_SIGS)


def _ptr(a):
    """data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(_vp)
    return _vp(a.data_ptr())


def _vec(t, n, what, dtype=None):
    """Device-vector argument check (before any pointer crosses the ABI): a
    contiguous CUDA tensor of the hot path's dtype (fp64 unless stated) with at
    least n entries.  Raises GmgError(GMG_E_INVALID_ARG) instead of letting a
    kernel read or write out of bounds."""
    import torch
    dtype = torch.float64 if dtype is None else dtype
    if not isinstance(t, torch.Tensor):
        raise GmgError(1, f"{what}: expected a torch CUDA tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise GmgError(1, f"{what}: tensor is on {t.device}, expected a CUDA device")
    if t.dtype != dtype:
        raise GmgError(1, f"{what}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise GmgError(1, f"{what}: tensor is not contiguous")
    if t.numel() < n:
        raise GmgError(1, f"{what}: {t.numel()} entries, expected {n}")
    return _vp(t.data_ptr())


def _stream(stream):
    if stream is not None:
        return _vp(stream)
    import torch
    return _vp(torch.cuda.current_stream().cuda_stream)


# ------------------------------------------------------------------ recipes
def recipe_from_config(cfg: dict, passes: int | None = -1) -> Recipe:
    """gmg_recipe from a gmg_inputs config dict (parameters only)."""
    r = Recipe()
    r.dim = cfg["dim"]
    r.n_trees = len(cfg["trees"])
    for t, pos in enumerate(cfg["trees"]):
        for j in range(cfg["dim"]):
            r.tree_xyz[3 * t + j] = pos[j]
    r.global_refinements = cfg["global_refinements"]
    rules = {"center_ball": 1, "sphere_surface": 2, "corner_dist": 3}
    r.rule = rules[cfg["rule"]]
    npass = cfg["passes"] if passes == -1 else passes
    r.n_passes = -1 if npass is None else int(npass)
    for j in range(3):
        r.center_den[j] = 1
    if "center" in cfg:
        for j, (n, d) in enumerate(cfg["center"]):
            r.center_num[j], r.center_den[j] = n, d
    if "radius" in cfg:
        r.radius_num, r.radius_den = cfg["radius"]
    else:
        r.radius_num, r.radius_den = 0, 1
    r.shell_num, r.shell_den = cfg.get("shell", (0, 1))
    if "corner" in cfg:
        for j, v in enumerate(cfg["corner"]):
            r.corner[j] = v
        r.s = cfg["s"]
        r.lmax = cfg["lmax"]
    return r


# ------------------------------------------------------------------ handles
class Forest:
    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:   # _lib is None at interpreter shutdown
            _lib.gmg_forest_destroy(self.h)
            self.h = None

    def info(self):
        d, t, n, L = C.c_int(), C.c_int(), C.c_int64(), C.c_int()
        _check(_lib.gmg_forest_info(self.h, C.byref(d), C.byref(t), C.byref(n), C.byref(L)))
        return dict(dim=d.value, n_trees=t.value, n_leaves=n.value, max_level=L.value)

    def count_nodes(self, k):
        """All leaf nodes of degree k (R22), without the level topology."""
        n = C.c_int64()
        _check(_lib.gmg_forest_count_nodes(self.h, k, C.byref(n)))
        return n.value

    def leaves(self):
        n = self.info()["n_leaves"]
        tree = np.empty(n, np.int32)
        lev = np.empty(n, np.int8)
        mor = np.empty(n, np.uint64)
        _check(_lib.gmg_export_leaves(self.h, _ptr(tree), _ptr(lev), _ptr(mor)))
        return tree, lev, mor


def gmg_forest_generate(recipe: Recipe) -> Forest:
    h = _vp()
    _check(_lib.gmg_forest_generate(C.byref(recipe), C.byref(h)))
    return Forest(h)


SEQUENCES = {"uniform": 0, "circle": 1, "quadrant": 2, "annulus": 3}


def gmg_forest_sequence(dim: int, kind: str, L: int) -> Forest:
    """The paper's partitioning-study mesh sequences, see gmg.h."""
    h = _vp()
    _check(_lib.gmg_forest_sequence(dim, SEQUENCES[kind], L, C.byref(h)))
    return Forest(h)


def gmg_forest_create(dim, trees, leaf_tree, leaf_level, leaf_morton, flags=0) -> Forest:
    t = np.ascontiguousarray(np.asarray(trees, dtype=np.int32).reshape(-1))
    lt = np.ascontiguousarray(leaf_tree, dtype=np.int32)
    ll = np.ascontiguousarray(leaf_level, dtype=np.int8)
    lm = np.ascontiguousarray(leaf_morton, dtype=np.uint64)
    h = _vp()
    _check(_lib.gmg_forest_create(dim, t.size // dim, _ptr(t), lt.size, _ptr(lt), _ptr(ll), _ptr(lm), flags,
                                  C.byref(h)))
    return Forest(h)


class Partitioning:
    def __init__(self, handle, forest, n_ranks):
        self.h = handle
        self.forest = forest      # keep the forest alive
        self.n_ranks = n_ranks

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:   # _lib is None at interpreter shutdown
            _lib.gmg_partition_destroy(self.h)
            self.h = None

    def model(self, W0_override=-1):
        m = Model()
        _check(_lib.gmg_partition_model(self.h, W0_override, C.byref(m)))
        nl = m.n_levels
        return dict(n_levels=nl, W_opt=(m.W_opt_num, m.W_opt_den), W_sync=m.W_sync, W=m.W,
                    eta=(m.eta_num, m.eta_den), N=list(m.N[:nl]), W_l=list(m.W_l[:nl]),
                    ghost_children=list(m.ghost_children[:nl]), children=list(m.children[:nl]))

    def tallies(self):
        nl = self.model()["n_levels"]
        out = np.empty(nl * self.n_ranks, np.int64)
        _check(_lib.gmg_export_tallies(self.h, _ptr(out)))
        return out.reshape(nl, self.n_ranks)

    def level_cells(self, level):
        n = C.c_int64()
        _check(_lib.gmg_export_level_cells(self.h, level, C.byref(n), None, None, None))
        key = np.empty(n.value, np.uint64)
        own = np.empty(n.value, np.int32)
        leaf = np.empty(n.value, np.uint8)
        _check(_lib.gmg_export_level_cells(self.h, level, C.byref(n), _ptr(key), _ptr(own), _ptr(leaf)))
        return key, own, leaf


PARTITION_MODES = {"first_child": 0, "per_level": 1}


def gmg_partition(forest: Forest, n_ranks: int, mode: str = "first_child", coarse_cells: int = 0) -> Partitioning:
    """SFC partition with the first-child rule or, mode="per_level",
    every level balanced on its own (P:597 alternative, reading R29);
    coarse_cells > 0 gathers the levels with at most that many cells on rank 0
    (gmg_partition_ex)."""
    h = _vp()
    _check(_lib.gmg_partition_ex(forest.h, n_ranks, PARTITION_MODES[mode], int(coarse_cells), C.byref(h)))
    return Partitioning(h, forest, n_ranks)


def gmg_params_default() -> Params:
    p = Params()
    _lib.gmg_params_default(C.byref(p))
    return p


class Hierarchy:
    """Owns a gmg_hierarchy.  Keeps the partition (and through it the forest),
    the coefficient array, the communicator and the allocator callbacks alive
    for as long as the hierarchy exists: the library holds raw pointers to them."""

    def __init__(self, handle, part, coef=None, comm=None, alloc=None):
        self.h = handle
        self.part = part
        self._coef = coef
        self.comm = comm
        self._alloc = alloc
        i = self.info()
        self.n_owned = i["n_owned"]
        self._dim, self._k = i["dim"], i["k"]
        self._level_dofs = i["level_dofs"]
        self._n_ranks = i["n_ranks"]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:   # _lib is None at interpreter shutdown
            _lib.gmg_hierarchy_destroy(self.h)
            self.h = None

    def close(self):
        """Destroy the hierarchy now (collective for multi-rank hierarchies)."""
        self.__del__()

    def _local_len(self, level):
        fo, no, gh = self.rank_level(level)
        return no + len(gh)

    def info(self) -> dict:
        i = Info()
        _check(_lib.gmg_hierarchy_info(self.h, C.byref(i)))
        nl = i.n_levels
        out = {f: getattr(i, f) for f, _ in Info._fields_ if not f.startswith("level_")}
        for f in ("level_dofs", "level_cells", "level_families", "level_S", "level_E", "level_B",
                  "level_leaf_cells", "level_r1", "level_gf"):
            out[f] = list(getattr(i, f)[:nl])
        return out

    # ---------- integer exports
    def level_dofs(self, level):
        n = C.c_int64()
        _check(_lib.gmg_export_level_dofs(self.h, level, C.byref(n), None, None, None, None))
        key = np.empty(n.value, np.uint64)
        cls = np.empty(n.value, np.uint8)
        own = np.empty(n.value, np.int32)
        can = np.empty(n.value, np.int64)
        _check(_lib.gmg_export_level_dofs(self.h, level, C.byref(n), _ptr(key), _ptr(cls), _ptr(own), _ptr(can)))
        return key, cls, own, can

    def leaf_dofs(self):
        n = C.c_int64()
        _check(_lib.gmg_export_leaf_dofs(self.h, C.byref(n), None, None, None, None))
        key = np.empty(n.value, np.uint64)
        lam = np.empty(n.value, np.int8)
        own = np.empty(n.value, np.int32)
        can = np.empty(n.value, np.int64)
        _check(_lib.gmg_export_leaf_dofs(self.h, C.byref(n), _ptr(key), _ptr(lam), _ptr(own), _ptr(can)))
        return key, lam, own, can

    def rank_level(self, level):
        """(first_owned, n_owned, ghost global indices) of this rank on `level`."""
        fo, no, ng = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.gmg_export_rank_level(self.h, level, C.byref(fo), C.byref(no), C.byref(ng), None))
        gh = np.empty(ng.value, np.int64)
        _check(_lib.gmg_export_rank_level(self.h, level, C.byref(fo), C.byref(no), C.byref(ng), _ptr(gh)))
        return fo.value, no.value, gh

    def local_level(self, level):
        """Rank-local layout in keys (gmg_export_local_level): dict of numpy arrays."""
        no, ng, npr = C.c_int64(), C.c_int64(), C.c_int32()
        _check(_lib.gmg_export_local_level(self.h, level, C.byref(no), C.byref(ng), None, None, None, C.byref(npr),
                                           None, None, None, None, None))
        ok = np.empty(no.value, np.uint64)
        gk = np.empty(ng.value, np.uint64)
        go = np.empty(ng.value, np.int32)
        peers = np.empty(npr.value, np.int32)
        so = np.empty(npr.value + 1, np.int64)
        ro = np.empty(npr.value + 1, np.int64)
        _check(_lib.gmg_export_local_level(self.h, level, C.byref(no), C.byref(ng), _ptr(ok), _ptr(gk), _ptr(go),
                                           C.byref(npr), _ptr(peers), _ptr(so), _ptr(ro), None, None))
        si = np.empty(int(so[-1]), np.int32)
        ri = np.empty(int(ro[-1]), np.int32)
        _check(_lib.gmg_export_local_level(self.h, level, C.byref(no), C.byref(ng), None, None, None, C.byref(npr),
                                           None, None, None, _ptr(si), _ptr(ri)))
        return dict(owned_key=ok, ghost_key=gk, ghost_owner=go, peers=peers, send_off=so, recv_off=ro,
                    send_idx=si, recv_idx=ri)

    def local_tables(self, level):
        """Local tables before device reordering (GMG_HOST_ONLY hierarchies)."""
        nc, nf = C.c_int64(), C.c_int64()
        _check(_lib.gmg_export_local_tables(self.h, level, C.byref(nc), C.byref(nf), None, None, None, None, None,
                                            None))
        lv = self.local_level(level)
        nloc = lv["owned_key"].size + lv["ghost_key"].size
        i = self.info()
        nn = (i["k"] + 1) ** i["dim"]
        row = (2 * i["k"] + 1) ** i["dim"] + nn
        cd = np.empty(nc.value * nn, np.int32)
        xf = np.empty(nf.value * row, np.int32)
        cls = np.empty(nloc, np.uint8)
        lam = np.empty(nloc, np.uint8)
        ev = np.empty(nloc, np.float64)
        cg = np.empty(nc.value, np.int64)
        _check(_lib.gmg_export_local_tables(self.h, level, C.byref(nc), C.byref(nf), _ptr(cd), _ptr(xf), _ptr(cls),
                                            _ptr(lam), _ptr(ev), _ptr(cg)))
        return dict(cell_dofs=cd.reshape(-1, nn), xfer=xf.reshape(-1, row) if nf.value else xf, cls=cls, lam=lam,
                    eig_v=ev, cell_global=cg)

    def owned_leaf_keys(self):
        """(keys, lambda) of this rank's free leaf DoFs in leaf order."""
        n = C.c_int64()
        _check(_lib.gmg_export_owned_leaf_keys(self.h, C.byref(n), None, None))
        k = np.empty(n.value, np.uint64)
        lam = np.empty(n.value, np.int8)
        _check(_lib.gmg_export_owned_leaf_keys(self.h, C.byref(n), _ptr(k), _ptr(lam)))
        return k, lam

    def cell_dofs(self, level):
        n = C.c_int64()
        _check(_lib.gmg_export_cell_dofs(self.h, level, C.byref(n), None))
        info = self.info()
        nn = (info["k"] + 1) ** info["dim"]
        out = np.empty(n.value * nn, np.int64)
        _check(_lib.gmg_export_cell_dofs(self.h, level, C.byref(n), _ptr(out)))
        return out.reshape(n.value, nn)

    # ---------- hot path (device tensors)
    def vcycle(self, b, x, stream=None):
        _check(_lib.gmg_vcycle(self.h, _vec(b, self.n_owned, "b"), _vec(x, self.n_owned, "x"), _stream(stream)))

    def solve_cg(self, b, x, rtol=1e-8, max_it=200, stream=None, raise_on_fail=True):
        it = C.c_int()
        rel = C.c_double()
        code = _lib.gmg_solve_cg(self.h, _vec(b, self.n_owned, "b"), _vec(x, self.n_owned, "x"), rtol, max_it,
                                 C.byref(it), C.byref(rel), _stream(stream))
        if code != GMG_OK and (raise_on_fail or code != 9):
            _check(code)
        return it.value, rel.value, code

    def rhs_constant(self, f, b, stream=None):
        _check(_lib.gmg_rhs_constant(self.h, f, _vec(b, self.n_owned, "b"), _stream(stream)))

    def level_apply(self, level, x, y, stream=None):
        n = self._level_dofs[level]
        _check(_lib.gmg_level_apply(self.h, level, _vec(x, n, "x"), _vec(y, n, "y"), _stream(stream)))

    def level_apply_kernel(self, level, x, y, stream=None):
        """Rank-local kernel only (timing); fp64 tensors, or fp32 tensors for the
        operator of the mixed-precision V-cycle."""
        import torch
        f32 = isinstance(x, torch.Tensor) and x.dtype == torch.float32
        fn = _lib.gmg_level_apply_kernel_f32 if f32 else _lib.gmg_level_apply_kernel
        n = self._local_len(level)
        dt = torch.float32 if f32 else torch.float64
        _check(fn(self.h, level, _vec(x, n, "x", dt), _vec(y, n, "y", dt), _stream(stream)))

    def restrict(self, level, r, dc, stream=None):
        _check(_lib.gmg_restrict(self.h, level, _vec(r, self._level_dofs[level], "r"),
                                 _vec(dc, self._level_dofs[level - 1] if level >= 1 else 0, "dc"), _stream(stream)))

    def prolongate(self, level, xc, xf, stream=None):
        _check(_lib.gmg_prolongate(self.h, level, _vec(xc, self._level_dofs[level - 1] if level >= 1 else 0, "xc"),
                                   _vec(xf, self._level_dofs[level], "xf"), _stream(stream)))

    def leaf_apply(self, u, v, stream=None):
        _check(_lib.gmg_leaf_apply(self.h, _vec(u, self.n_owned, "u"), _vec(v, self.n_owned, "v"), _stream(stream)))

    def level_smooth(self, level, g, x, x_is_zero, stream=None):
        n = self._level_dofs[level]
        _check(_lib.gmg_level_smooth(self.h, level, _vec(g, n, "g"), _vec(x, n, "x"), int(bool(x_is_zero)),
                                     _stream(stream)))

    def level_diagonal(self, level, diag, stream=None):
        _check(_lib.gmg_level_diagonal(self.h, level, _vec(diag, self._level_dofs[level], "diag"), _stream(stream)))

    def coarse_chebyshev(self):
        """(lambda_min, lambda_max, degree) of the Chebyshev coarse solver (degree 0: Cholesky)."""
        lo, hi, m = C.c_double(), C.c_double(), C.c_int()
        _check(_lib.gmg_get_coarse_chebyshev(self.h, C.byref(lo), C.byref(hi), C.byref(m)))
        return lo.value, hi.value, m.value

    def get_eigen(self, level):
        v = C.c_double()
        _check(_lib.gmg_get_eigen(self.h, level, C.byref(v)))
        return v.value

    def set_eigen(self, level, lam):
        _check(_lib.gmg_set_eigen(self.h, level, float(lam)))

    def profile_vcycle(self, b, x, n_rep=3, stream=None):
        """Per (kernel kind, level) launch statistics of n_rep eager V-cycles
        (gmg_profile_vcycle): dicts with kind, level, launches, seconds (summed),
        bytes and bytes_layout per launch."""
        cap = 4096
        arr = (KernelStat * cap)()
        n = C.c_int()
        _check(_lib.gmg_profile_vcycle(self.h, _vec(b, self.n_owned, "b"), _vec(x, self.n_owned, "x"), int(n_rep),
                                       arr, cap, C.byref(n), _stream(stream)))
        return [dict(kind=KERNEL_KINDS[a.kind], level=a.level, launches=a.launches, seconds=a.seconds,
                     bytes=a.bytes, bytes_layout=a.bytes_layout) for a in arr[:min(n.value, cap)]]

    def launch_count(self):
        v = C.c_int64()
        _check(_lib.gmg_launch_count(self.h, C.byref(v)))
        return v.value

    def launch_profile(self):
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.gmg_launch_profile(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


class LocalWorld:
    """n ranks as host threads of one process (test transport, gmg_local_world)."""

    def __init__(self, n):
        self.h = _vp()
        _check(_lib.gmg_local_world_create(n, C.byref(self.h)))
        self.n = n

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:   # _lib is None at interpreter shutdown
            _lib.gmg_local_world_destroy(self.h)
            self.h = None


class HostWorld:
    """Ranks as separate processes joined through POSIX shared memory
    (gmg_host_world, host-staged exchanges; the multi-process path on a machine
    with fewer GPUs than ranks).  Collective create and destroy."""

    def __init__(self, name: str, n_ranks: int, rank: int, slot_bytes: int = 256 << 20):
        self.h = _vp()
        _check(_lib.gmg_host_world_create(name.encode(), n_ranks, rank, slot_bytes, C.byref(self.h)))
        self.n, self.rank = n_ranks, rank

    def destroy(self):
        if getattr(self, "h", None):
            _check(_lib.gmg_host_world_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def torch_allocator(device: int | None = None):
    """(dev_alloc, dev_free) ctypes callbacks over the torch caching allocator
    (gmg_params.dev_alloc / dev_free).  Keep the returned pair alive as long as
    the hierarchy (Hierarchy does)."""
    import torch

    dev = torch.cuda.current_device() if device is None or device < 0 else device

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), dev, 0)
        except Exception:
            return None

    def _free(ptr, nbytes, stream, ctx):
        torch.cuda.caching_allocator_delete(ptr)

    return DEV_ALLOC(_alloc), DEV_FREE(_free)


def gmg_nccl_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.gmg_nccl_get_unique_id(buf))
    return buf.raw


class NcclComm:
    def __init__(self, uid: bytes, n_ranks: int, rank: int):
        self.h = _vp()
        _check(_lib.gmg_nccl_comm_init(C.create_string_buffer(uid, 128), n_ranks, rank, C.byref(self.h)))

    def destroy(self):
        if getattr(self, "h", None) and _lib is not None:   # _lib is None at interpreter shutdown
            _lib.gmg_nccl_comm_destroy(self.h)
            self.h = None


def gmg_setup(forest: Forest, part: Partitioning, k=2, host_only=False, cheb_degree=4, rank=0,
              coef_level2=None, graph=True, device=-1, comm=None, mixed=False,
              coarse="cholesky", allocator=None, rank_local=False, eig_key=False) -> Hierarchy:
    """comm: None (one rank), a LocalWorld (ranks as threads), a HostWorld (ranks
    as processes, host-staged) or an NcclComm.  allocator: None (cudaMalloc) or
    "torch" (the torch caching allocator through gmg_params.dev_alloc/dev_free)."""
    p = gmg_params_default()
    p.k = k
    p.cheb_degree = cheb_degree
    p.rank = rank
    p.n_ranks = part.n_ranks
    p.device = device
    p.flags = (GMG_HOST_ONLY if host_only else 0) | (0 if graph else GMG_NO_GRAPH) | \
        (GMG_MIXED_PRECISION if mixed else 0) | (GMG_RANK_LOCAL if rank_local else 0) | \
        (GMG_EIG_KEY if eig_key else 0)
    p.coarse_solver = {"cholesky": 0, "chebyshev": 1}[coarse]
    if isinstance(comm, LocalWorld):
        p.flags |= GMG_LOCAL_RANKS
        p.nccl_comm = comm.h
    elif isinstance(comm, HostWorld):
        p.flags |= GMG_HOST_RANKS
        p.nccl_comm = comm.h
    elif comm is not None:
        p.nccl_comm = comm.h
    coef = None
    if coef_level2 is not None:
        coef = np.ascontiguousarray(coef_level2, dtype=np.float64)
        p.coef_level2 = coef.ctypes.data_as(C.POINTER(C.c_double))
    alloc = None
    if allocator == "torch" and not host_only:
        alloc = torch_allocator(device)
        p.dev_alloc, p.dev_free = alloc
    elif allocator not in (None, "cuda", "torch"):
        raise ValueError(f"allocator {allocator!r}")
    h = _vp()
    _check(_lib.gmg_setup(forest.h, part.h, C.byref(p), C.byref(h)))
    return Hierarchy(h, part, coef, comm=comm, alloc=alloc)


def build_config(cfg: dict, n_ranks=1, host_only=False, passes=-1, **kw):
    """Forest -> partition -> hierarchy for a gmg_inputs config dict."""
    f = gmg_forest_generate(recipe_from_config(cfg, passes))
    part = gmg_partition(f, n_ranks)
    h = gmg_setup(f, part, k=cfg["k"], host_only=host_only, **kw)
    return f, part, h
