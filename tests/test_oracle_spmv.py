"""The oracle's multi-threaded CSR matvec (oracle/_spmv.c, used only to time the
oracle on all host cores) gives bit-identical results to scipy's single-thread
product, so the oracle's values do not depend on the thread count."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import spmv, forest as F, mg
from gmg_inputs import config, uniform_pm1


@pytest.fixture(scope="module", autouse=True)
def built():
    spmv.build()
    yield
    spmv.set_threads(1)


@pytest.mark.parametrize("idx", ["int32", "int64"])
def test_matvec_bit_identical(idx):
    rng = np.random.default_rng(4)
    A = sp.random(3000, 3000, density=0.01, random_state=5, format="csr")
    A.indptr = A.indptr.astype(idx)
    A.indices = A.indices.astype(idx)
    x = rng.standard_normal(3000)
    assert spmv.set_threads(4) == 4
    y = spmv.mv(A, x)
    spmv.set_threads(1)
    assert np.array_equal(y, A @ x)


def test_vcycle_independent_of_threads():
    cfg = config("c3")
    h = mg.build(F.generate(cfg, passes=2), cfg["k"])
    b = uniform_pm1(h.leaf.n_free)
    spmv.set_threads(1)
    x1 = mg.vcycle(h, b)
    spmv.set_threads(4)
    x4 = mg.vcycle(h, b)
    spmv.set_threads(1)
    assert np.array_equal(x1, x4)
