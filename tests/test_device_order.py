"""Integer pin of the device order (csrc/plan.hpp): on every level the tensor
kernels run (3D, levels >= 1, no per-cell coefficients inside a family), R1 =
the rows exactly one executed patch touches (one rank: no row is needed
remotely).  A patch is a family (2^d consecutive cells, children of one parent,
SFC order) or, for Q2, a complete grandfamily: 8 consecutive families whose
parents are children 0..7 of one level-(l-2) cell and share one coefficient
(config 4: levels >= 4, where all 64 cells inherit one level-2 ancestor).  The
count is recomputed here from the exported cell->DoF table and the level cell
keys: a row's touch count is the number of distinct patches among the cells
containing it; the number of grandfamilies must equal gmg_info.level_gf.
Bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1904_03317_b200 as G  # noqa: E402
from gmg_inputs import config, log_uniform_coef  # noqa: E402

CASES = [("c3", 4, {}), ("c3", 4, {"k": 1}), ("c4", -1, {"s": 2, "lmax": 7})]


def touch_counts(cd, n, nch, patch_of_family):
    fam = np.repeat(np.arange(len(cd)) // nch, cd.shape[1])
    patch = patch_of_family[fam]
    dof = cd.ravel()
    ok = dof >= 0
    pairs = np.unique(np.stack([dof[ok], patch[ok]], 1), axis=0)   # (row, patch) once each
    return np.bincount(pairs[:, 0], minlength=n)


def patches(keys, nch, use_gf):
    """patch id per family: grandfamilies (8 consecutive families with parents
    k0|0 .. k0|7) or the family itself; and the number of grandfamilies"""
    pk = keys[::nch] >> np.uint64(3)            # parent key of each family
    nf = pk.size
    pid = np.arange(nf)
    ngf = 0
    f = 0
    while use_gf and f + 7 < nf:
        k0 = int(pk[f])
        if k0 & 7 == 0 and all(int(pk[f + j]) == (k0 | j) for j in range(8)):
            pid[f:f + 8] = nf + ngf
            ngf += 1
            f += 8
        else:
            f += 1
    return pid, ngf


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
        keys = h.part.level_cells(l)[0]
        use_gf = tensor and info["k"] == 2 and l >= 2 and (coef is None or l >= 4) and l > info["small_levels"]
        pid, ngf = patches(keys, nch, use_gf)
        assert info["level_gf"][l] == ngf, (l, info["level_gf"][l], ngf)
        expect = int((touch_counts(h.cell_dofs(l), n, nch, pid) == 1).sum()) if tensor and n else 0
        assert info["level_r1"][l] == expect, (l, info["level_r1"][l], expect)
    assert sum(info["level_r1"]) > 0
