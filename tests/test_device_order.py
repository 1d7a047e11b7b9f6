"""Integer pin of the device order (csrc/plan.hpp): on every level the
family-tensor kernel runs (3D, levels >= 1, no per-cell coefficients inside a
family), R1 = the rows exactly one family patch touches (one rank: no row is
needed remotely).  The count is recomputed here from the exported cell->DoF
table: a family is 2^d consecutive cells of the level (children of one parent,
SFC order), and a row's touch count is the number of distinct families among
the cells that contain it.  Bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, log_uniform_coef  # noqa: E402

CASES = [("c3", 4, {}), ("c3", 4, {"k": 1}), ("c4", -1, {"s": 2, "lmax": 7})]


def touch_counts(cd, n, nch):
    fam = np.repeat(np.arange(len(cd)) // nch, cd.shape[1])
    dof = cd.ravel()
    ok = dof >= 0
    pairs = np.unique(np.stack([dof[ok], fam[ok]], 1), axis=0)   # (row, family) once each
    return np.bincount(pairs[:, 0], minlength=n)


@pytest.mark.parametrize("name,passes,over", CASES, ids=["c3p4", "c3p4-k1", "c4s"])
def test_r1_is_rows_touched_by_one_family(name, passes, over):
    cfg = dict(config(name))
    cfg.update(over)
    coef = log_uniform_coef(4 ** cfg["dim"] * len(cfg["trees"])) if cfg.get("coef") else None
    _, _, h = G.build_config(cfg, passes=passes, coef_level2=coef)
    info = h.info()
    nch = 2 ** info["dim"]
    assert info["level_r1"][0] == 0
    for l in range(1, info["n_levels"]):
        n = info["level_dofs"][l]
        tensor = info["dim"] == 3 and not (coef is not None and l <= 2)   # R15: levels 0-2 carry per-cell data
        expect = int((touch_counts(h.cell_dofs(l), n, nch) == 1).sum()) if tensor and n else 0
        assert info["level_r1"][l] == expect, (l, info["level_r1"][l], expect)
    assert sum(info["level_r1"]) > 0
