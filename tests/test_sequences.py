"""Partition-efficiency and communication-ratio study (
PAPER.md §3.5-3.6, Figs. 3-5).

1. The mesh sequences uniform / circle / quadrant / annulus (reading
   R27: one coarse cell = [-1,1]^d) built by the library equal the oracle's
   independent construction leaf by leaf, and the partition model (W_opt,
   W_sync, W, eta, ghost children) is bit-exact against the oracle.
2. Pins from the paper's prose (the figures themselves are not in the
   container), at desk scale with SPEC.md acceptance tolerances:
   uniform "100% efficiency"; annulus "saturation ... about 30%"
    reached for p >= 64 in 2D; circle "very high efficiency ... from
   the beginning, then dropping off"; "in all cases, the efficiency
   stays above 30%" while cells per processor >= 1000; ghost
   children "less than 1%" of the children at the paper's scale, growing
   sublinearly in p (desk-scale bound < 5%).
   The quadrant's plateau "saturation ... with 60% for the quadrant ... only
   begins dropping again when the problem size is down to less than 1000 cells
   per processor (seen only in the quadrant case)" IS reproduced
   under reading R27 once p reaches ~10^3: eta ~0.57 flat from p = 1024 to
   8192 at L = 12/13, dropping below ~1000 cells per rank (round 1 stopped the
   sweep at p = 256, where eta is still 0.78).
"""
from fractions import Fraction

import numpy as np
import pytest

import paper_1904_03317_b200 as G
from oracle import forest as F, partition as Pt
from test_parity_integer import compare_forest, compare_partition

SMALL = [("uniform", 2, 4), ("circle", 2, 7), ("quadrant", 2, 6), ("annulus", 2, 8),
         ("uniform", 3, 3), ("circle", 3, 4), ("quadrant", 3, 4), ("annulus", 3, 5)]


@pytest.mark.parametrize("kind,d,L", SMALL, ids=[f"{k}{d}d-L{L}" for k, d, L in SMALL])
def test_sequence_equals_oracle(kind, d, L):
    of = F.sequence(d, kind, L)
    lf = G.gmg_forest_sequence(d, kind, L)
    compare_forest(lf, of)
    assert of.max_level == L or kind == "annulus"
    for p in (1, 3, 8, 16):
        compare_partition(G.gmg_partition(lf, p), of, p)


def test_sequence_closed_forms():
    # uniform: 4^L / 8^L leaves; quadrant 2D L=3: 28 leaves (one quadrant refined
    # twice, the three level-1 cells closed once); annulus needs L >= 4
    assert G.gmg_forest_sequence(2, "uniform", 5).info()["n_leaves"] == 4 ** 5
    assert G.gmg_forest_sequence(3, "uniform", 3).info()["n_leaves"] == 8 ** 3
    assert G.gmg_forest_sequence(2, "quadrant", 3).info()["n_leaves"] == 28
    with pytest.raises(G.GmgError):
        G.gmg_forest_sequence(2, "annulus", 3)


def _eta_ratio(f, p):
    m = G.gmg_partition(f, p).model()
    eta = Fraction(*m["eta"])
    ratio = sum(m["ghost_children"]) / max(sum(m["children"]), 1)
    return float(eta), ratio


def test_uniform_efficiency_100_percent():
    for p, L in ((4, 6), (16, 7), (64, 8)):            # >= 1000 leaves per rank
        eta, _ = _eta_ratio(G.gmg_forest_sequence(2, "uniform", L), p)
        assert eta >= 0.99, (p, L, eta)


def test_annulus_plateau_about_30_percent():
    f2 = G.gmg_forest_sequence(2, "annulus", 10)
    e2 = [_eta_ratio(f2, p)[0] for p in (16, 32, 64, 128, 256)]
    assert all(a >= b - 1e-12 for a, b in zip(e2, e2[1:])), e2      # drops, then saturates
    assert all(0.20 <= e <= 0.40 for e in e2[2:]), e2
    f3 = G.gmg_forest_sequence(3, "annulus", 7)
    e3 = [_eta_ratio(f3, p)[0] for p in (16, 32, 64, 128)]
    assert all(a >= b - 1e-12 for a, b in zip(e3, e3[1:])), e3
    assert 0.20 <= e3[-1] <= 0.40, e3


def test_circle_high_then_dropping():
    f = G.gmg_forest_sequence(2, "circle", 12)
    e = [_eta_ratio(f, p)[0] for p in (4, 16, 64, 256)]
    assert e[0] >= 0.99 and e[1] >= 0.9, e
    assert all(a >= b - 1e-12 for a, b in zip(e, e[1:])), e


def test_efficiency_above_30_percent_with_1000_cells_per_rank():
    cases = [("quadrant", 2, 12, (16, 64, 256)), ("annulus", 2, 10, (16, 64)), ("circle", 2, 12, (16, 64)),
             ("annulus", 3, 7, (16,)), ("quadrant", 3, 7, (8, 64, 256))]
    for kind, d, L, ps in cases:
        f = G.gmg_forest_sequence(d, kind, L)
        n = f.info()["n_leaves"]
        for p in ps:
            assert n / p >= 1000
            eta, _ = _eta_ratio(f, p)
            assert eta >= 0.30, (kind, d, L, p, eta)


def test_ghost_children_ratio_small_and_sublinear():
    f = G.gmg_forest_sequence(2, "annulus", 9)
    _, r16 = _eta_ratio(f, 16)
    _, r64 = _eta_ratio(f, 64)
    assert r64 < 0.05 and r64 < 4 * r16, (r16, r64)
    # larger problem, same p: the ratio shrinks (surface / volume)
    _, r64_big = _eta_ratio(G.gmg_forest_sequence(2, "annulus", 12), 64)
    assert r64_big < r64


def test_config3_partition_model_matches_survey_values():
    """Exact first-child model on the full config-3 forest (5.3M leaves) against the
    values SURVEY §8(c.3) lists (independent computation): eta at p = 1/2/4/8,
    W = W_sync, one octant of level-10 cells per rank at p = 8."""
    import json
    import os
    from gmg_inputs import config
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config_counts.json")))
    c3 = gold["c3_partition"]
    lf = G.gmg_forest_generate(G.recipe_from_config(config("c3")))
    for p, eta in c3["eta"].items():
        part = G.gmg_partition(lf, int(p))
        m = part.model()
        assert Fraction(*m["eta"]) == Fraction(*eta), p
        assert m["N"] == gold["c3"]["N_l"]
        if p in c3["W"]:
            assert m["W"] == c3["W"][p] == m["W_sync"]
        if p == "8":
            t = part.tallies()
            assert list(t[10]) == [c3["p8_level10_cells_per_rank"]] * 8


def test_quadrant_plateau_about_60_percent():
    """the quadrant's efficiency drops, then saturates near 60% over a
    wide range of processor counts and drops again below ~1000 cells per rank."""
    f = G.gmg_forest_sequence(2, "quadrant", 12)
    n = f.info()["n_leaves"]
    ps = (64, 256, 1024, 2048, 4096, 16384)
    e = [_eta_ratio(f, p)[0] for p in ps]
    assert all(a >= b - 1e-12 for a, b in zip(e, e[1:])), e            # never rises
    plateau = e[2:5]                                                       # p = 1024 .. 4096 (>= 1000 cells/rank)
    assert all(n / p >= 1000 for p in ps[2:5])
    assert all(0.50 <= x <= 0.65 for x in plateau), plateau
    assert max(plateau) - min(plateau) <= 0.02, plateau                   # flat
    assert e[1] - e[2] > 0.1                                               # reached after a drop
    assert n / ps[-1] < 1000 and e[-1] < min(plateau) - 0.02              # drops again below 1000 cells/rank
