"""CSR matvec dispatch for the oracle (TEST INFRASTRUCTURE ONLY).

``mv(A, x)`` is ``A @ x`` (scipy, one thread) unless ``set_threads(n > 1)`` was
called and ``oracle/_spmv.so`` (built by ``__graft_entry__.build()``) loads; then
the same product runs row-parallel in C with the row sums in scipy's order, so
the oracle's results do not depend on the thread count (bit-identical).  Only
the timing of the reported CPU baseline uses more than one thread."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_spmv.so")
_lib = None
_threads = 1


def build(quiet: bool = True) -> str:
    """gcc -O2 -fopenmp -ffp-contract=off -shared oracle/_spmv.c -> oracle/_spmv.so"""
    import subprocess
    src = os.path.join(_HERE, "_spmv.c")
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", src, "-o", _SO],
                   check=True, capture_output=quiet)
    return _SO


def _load():
    global _lib
    if _lib is None and os.path.exists(_SO):
        lib = C.CDLL(_SO)
        for nm, it in (("csr_matvec_i32", C.c_int32), ("csr_matvec_i64", C.c_int64)):
            f = getattr(lib, nm)
            f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
            f.restype = None
        lib.spmv_max_threads.restype = C.c_int
        _lib = lib
    return _lib


def set_threads(n: int) -> int:
    """Threads for mv(); returns the number actually used (1 without _spmv.so)."""
    global _threads
    _threads = max(1, int(n))
    if _threads > 1 and _load() is None:
        _threads = 1
    return _threads


def threads() -> int:
    return _threads


def mv(A, x: np.ndarray) -> np.ndarray:
    if _threads <= 1 or not sp.isspmatrix_csr(A) or A.dtype != np.float64 or x.dtype != np.float64:
        return A @ x
    lib = _load()
    x = np.ascontiguousarray(x)
    y = np.empty(A.shape[0])
    fn = lib.csr_matvec_i32 if A.indptr.dtype == np.int32 else lib.csr_matvec_i64
    ip = np.ascontiguousarray(A.indptr)
    ix = np.ascontiguousarray(A.indices, dtype=ip.dtype)
    fn(A.shape[0], ip.ctypes.data, ix.ctypes.data, A.data.ctypes.data, x.ctypes.data, y.ctypes.data, _threads)
    return y
