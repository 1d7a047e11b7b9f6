"""The plain operator's column kernel (kernels.cuh fam_col_apply, GMG_COL = 16 / 32
families per block) (opt-in; slower than the default)
against fam_tensor_apply<TA_APPLY> (GMG_COL=0): the same
Kronecker sum on the same family patches in another summation order, so level
applies and V-cycles agree to 1e-13 relative in fp64 (2e-6 for the fp32 V-cycle)
and CG takes the same iterations.  The oracle comparison of the default path is
tests/test_gpu_parity.py.  Each variant runs in its own process (GMG_COL is read
once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from test_grandfamily import ROOT, SCRIPT

pytestmark = pytest.mark.gpu

CASES = [("c3", 4, {}, False), ("c4", -1, {"s": 2, "lmax": 7}, True), ("c3", 3, {"k": 1}, False)]


def _run(tmp_path, name, passes, over, mixed, col):
    out = str(tmp_path / f"c{col}.npz")
    code = SCRIPT.format(root=ROOT, name=name, over=over, passes=passes, mixed=mixed, out=out)
    env = dict(os.environ, GMG_COL=col)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("name,passes,over,mixed", CASES, ids=["c3p4", "c4s-mixed", "c3p3-q1"])
def test_column_kernel_matches_tensor_kernel(tmp_path, name, passes, over, mixed):
    ref = _run(tmp_path, name, passes, over, mixed, "0")
    tol = 2e-6 if mixed else 1e-13
    for col in ("16", "32"):
        got = _run(tmp_path, name, passes, over, mixed, col)
        for key in ("y", "x"):
            a, b = got[key], ref[key]
            assert np.abs(a - b).max() <= tol * np.abs(b).max(), (col, key, np.abs(a - b).max() / np.abs(b).max())
        assert abs(int(got["it"]) - int(ref["it"])) <= (1 if mixed else 0)
