"""Rank-local topology (GMG_RANK_LOCAL, csrc/local_direct.cpp): each rank builds
only its families, the families of the parents of its next-finer families and
their vertex neighbours (only the mesh parts relevant to a processor
are stored; ownership is available without global communication).  It must
produce exactly the rank-local layout the global numbering yields (make_local):
owned/ghost keys and order, ghost owners, exchange plans, cell and transfer
tables in local indices, classes, lambda slots, the key-based eigen start vector
(R10b) and the leaf DoFs -- for every rank, both partition rules, 2D and 3D,
Q1 and Q2.  CPU only (GMG_HOST_ONLY)."""
import numpy as np
import pytest

import paper_1904_03317_b200 as G
from gmg_inputs import config

CASES = [("c1", 1, "first_child", (1, 2, 5)), ("c1", 2, "first_child", (3, 8)),
         ("c3p2", 2, "first_child", (1, 2, 3, 8)), ("c3p2", 1, "first_child", (4, 7)),
         ("c3p2", 2, "per_level", (3, 6)), ("c4s", 2, "first_child", (2, 5)), ("c4s", 2, "per_level", (4,)),
         ("brick8", 2, "first_child", (3, 5)), ("brick8", 1, "per_level", (5,)), ("c2p", 2, "first_child", (3,))]


def _cfg(name):
    if name == "c4s":
        cfg = config("c4")
        cfg.update(s=2, lmax=7)
        return cfg, -1
    if name == "c3p2":
        return config("c3"), 2
    if name == "c2p":                          # the L-shape config at a small depth
        cfg = config("c2")
        cfg.update(lmax=7)
        return cfg, -1
    return config(name), -1


@pytest.mark.parametrize("name,k,mode,ps,coarse", [c + (0,) for c in CASES] +
                         [("c3p2", 2, "first_child", (3, 8), 600), ("c4s", 2, "per_level", (4,), 100)])
def test_rank_local_equals_global_layout(name, k, mode, ps, coarse):
    cfg, passes = _cfg(name)
    f = G.gmg_forest_generate(G.recipe_from_config(cfg, passes))
    for p in ps:
        part = G.gmg_partition(f, p, mode=mode, coarse_cells=coarse)
        for r in range(p):
            hg = G.gmg_setup(f, part, k=k, rank=r, host_only=True, eig_key=True)
            hl = G.gmg_setup(f, part, k=k, rank=r, host_only=True, rank_local=True)
            n_levels = hg.info()["n_levels"]
            for l in range(n_levels):
                a, b = hg.local_level(l), hl.local_level(l)
                for key in a:
                    assert np.array_equal(a[key], b[key]), (p, r, l, key)
                ta, tb = hg.local_tables(l), hl.local_tables(l)
                for key in ta:
                    assert np.array_equal(ta[key], tb[key]), (p, r, l, key)
            ka, kb = hg.owned_leaf_keys(), hl.owned_leaf_keys()
            assert np.array_equal(ka[0], kb[0]) and np.array_equal(ka[1], kb[1]), (p, r)


def test_rank_local_single_rank_sizes():
    """With one rank the summed counts are the global sizes of the global build."""
    cfg = config("c3")
    f = G.gmg_forest_generate(G.recipe_from_config(cfg, 2))
    part = G.gmg_partition(f, 1)
    ig = G.gmg_setup(f, part, k=2, host_only=True).info()
    il = G.gmg_setup(f, part, k=2, host_only=True, rank_local=True).info()
    for key in ("n_leaf_nodes", "n_leaf_free", "n_leaf_hanging", "n_leaf_dirichlet", "n_owned", "first_owned",
                "level_dofs", "level_cells", "level_families", "level_S", "level_E", "level_B", "level_leaf_cells"):
        assert ig[key] == il[key], key


def test_rank_local_global_exports_refused():
    cfg = config("c1")
    f = G.gmg_forest_generate(G.recipe_from_config(cfg))
    part = G.gmg_partition(f, 2)
    h = G.gmg_setup(f, part, k=1, rank=1, host_only=True, rank_local=True)
    with pytest.raises(G.GmgError):
        h.level_dofs(1)
    with pytest.raises(G.GmgError):
        h.leaf_dofs()


# ------------------------------------------------------------------ gloo, world size 2 and 3
def _plan_worker(rank, world, port, name, coarse, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg, passes = _cfg(name)
        f = G.gmg_forest_generate(G.recipe_from_config(cfg, passes))
        part = G.gmg_partition(f, world, coarse_cells=coarse)
        h = G.gmg_setup(f, part, k=cfg["k"], rank=rank, host_only=True, rank_local=True)
        mine = []
        for l in range(h.info()["n_levels"]):
            lv = h.local_level(l)
            sends = {}
            for i, peer in enumerate(lv["peers"]):
                idx = lv["send_idx"][lv["send_off"][i]:lv["send_off"][i + 1]]
                sends[int(peer)] = lv["owned_key"][idx].tolist()
            recvs = {}
            for i, peer in enumerate(lv["peers"]):
                idx = lv["recv_idx"][lv["recv_off"][i]:lv["recv_off"][i + 1]] - lv["owned_key"].size
                recvs[int(peer)] = lv["ghost_key"][idx].tolist()
                assert (lv["ghost_owner"][idx] == peer).all()
            mine.append((sends, recvs, lv["owned_key"].tolist()))
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        # the plans of every pair match key by key, and no DoF is owned twice
        for l in range(len(mine)):
            for r in range(world):
                for peer, keys in allv[r][l][0].items():
                    assert allv[peer][l][1].get(r, []) == keys, (l, r, peer)
                for peer, keys in allv[r][l][1].items():
                    assert allv[peer][l][0].get(r, []) == keys, (l, r, peer)
            owned = [k for r in range(world) for k in allv[r][l][2]]
            assert len(owned) == len(set(owned))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("name,world,coarse", [("c3p2", 2, 0), ("c4s", 3, 0), ("c3p2", 3, 600)])
def test_gloo_rank_local_exchange_plans_match(name, world, coarse):
    """Each rank builds only its own part (rank-local); over gloo the ranks check
    that what r sends to q is, key by key and in order, what q expects from r, and
    that the owned sets are disjoint."""
    import multiprocessing as mp
    import socket
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ps = [ctx.Process(target=_plan_worker, args=(r, world, port, name, coarse, q)) for r in range(world)]
    for p_ in ps:
        p_.start()
    res = [q.get(timeout=300) for _ in ps]
    for p_ in ps:
        p_.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res


def test_rank_local_chunked_occurrence_sort(monkeypatch):
    """The rank-local builder sorts the halo's node occurrences in key-range chunks
    (bounded memory for config 5); forcing tiny chunks must give the same layout."""
    cfg, passes = _cfg("c3p2")
    f = G.gmg_forest_generate(G.recipe_from_config(cfg, passes))
    part = G.gmg_partition(f, 3)
    ref = [G.gmg_setup(f, part, k=2, rank=r, host_only=True, rank_local=True) for r in range(3)]
    monkeypatch.setenv("GMG_OCC_CHUNK", "1000")
    for r in range(3):
        h = G.gmg_setup(f, part, k=2, rank=r, host_only=True, rank_local=True)
        for l in range(h.info()["n_levels"]):
            a, b = ref[r].local_level(l), h.local_level(l)
            for key in a:
                assert np.array_equal(a[key], b[key]), (r, l, key)
            ta, tb = ref[r].local_tables(l), h.local_tables(l)
            for key in ta:
                assert np.array_equal(ta[key], tb[key]), (r, l, key)
