"""Planner parity (CPU): the library's plan lists must equal the oracle's
bit-exactly, and its volume statistics must equal the
oracle's closed forms (Eqs. 1-3, 10-11).

The library runs in loopback mode with SHIRO_F_HOST_ONLY: the same C++
planner (Hopcroft-Karp + König) as the distributed path, all virtual ranks in
one process, no device.  The oracle uses Dinic on the textbook flow network;
agreement is the canonical-cut uniqueness of DESIGN.md R1/R16."""
import numpy as np
import pytest

import oracle
import paper_2512_20178_b200 as sh
import shiro_gen
from conftest import random_csr

KINDS = ((sh.LIST_SEND_B, "send_b", False), (sh.LIST_SEND_C, "send_c", False),
         (sh.LIST_RECV_B, "send_b", True), (sh.LIST_RECV_C, "send_c", True))


def assert_lists_equal(pl, op, P):
    empty = np.empty(0, np.int64)
    for r in range(P):
        v = pl.rank_view(r)
        for p in range(P):
            if p == r:
                continue
            for kind, attr, recv in KINDS:
                key = (p, r) if recv else (r, p)
                got = v.list(p, kind)
                exp = getattr(op, attr).get(key, empty)
                assert np.array_equal(got, exp), (r, p, kind, got[:8], exp[:8])


def assert_stats_equal(pl, op, N, g=1):
    info = pl.info()
    vol = oracle.volumes(op, N)
    assert info["g_joint_rows"] == vol["joint_rows"]
    assert info["g_col_rows"] == vol["col_rows"]
    assert info["g_row_rows"] == vol["row_rows"]
    assert info["g_block_rows"] == vol["block_rows"]
    assert info["g_oblivious_rows"] == vol["oblivious_rows"]
    assert info["g_setup_bytes"] == vol["setup_bytes"]
    if g > 1:
        tt = oracle.tier_traffic(oracle.plan_hier(op, g), 1, 1)
        assert info["g_hier_inter_rows"] == tt["inter_rows"]
        assert info["g_hier_intra_rows"] == tt["intra_rows"]
        assert info["g_flat_inter_rows"] == oracle.flat_inter_rows(op, g)


FLAGS = {("joint", "rowmax"): 0, ("joint", "colmax"): sh.F_COVER_COLMAX,
         ("col", "rowmax"): sh.F_MODE_COL, ("row", "rowmax"): sh.F_MODE_ROW,
         ("block", "rowmax"): sh.F_MODE_BLOCK}


@pytest.mark.parametrize("seed", range(40))
def test_random_matrices(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 300))
    P = [1, 2, 3, 4, 8][seed % 5]
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.003, 0.2)), symmetric=seed % 3 == 0)
    part = oracle.uniform_partition(n, P)
    mode, rule = list(FLAGS)[seed % 5]
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 16, flags=FLAGS[(mode, rule)] | sh.F_HOST_ONLY)
    op = oracle.plan_flat(n, part, row_ptr, col, mode=mode, rule=rule)
    assert_lists_equal(pl, op, P)
    assert_stats_equal(pl, op, 16)


def test_uneven_and_empty_partitions():
    rng = np.random.default_rng(3)
    n = 50
    row_ptr, col, val = random_csr(rng, n, 0.1)
    for part in ([0, 0, 10, 10, 50], [0, 49, 50], [0, 1, 2, 3, 4, 50, 50, 50, 50]):
        part = np.array(part, np.int64)
        P = part.size - 1
        pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 8, flags=sh.F_HOST_ONLY)
        op = oracle.plan_flat(n, part, row_ptr, col)
        assert_lists_equal(pl, op, P)
        assert_stats_equal(pl, op, 8)


@pytest.mark.parametrize("P,g", [(4, 2), (8, 2), (8, 4)])
def test_hier_stats(P, g):
    rng = np.random.default_rng(P * 7 + g)
    n = 200
    row_ptr, col, val = random_csr(rng, n, 0.04, symmetric=True)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 32, group_size=g, flags=sh.F_HOST_ONLY)
    op = oracle.plan_flat(n, part, row_ptr, col)
    assert_lists_equal(pl, op, P)
    assert_stats_equal(pl, op, 32, g)


@pytest.mark.parametrize("cfg,P", [("c1", 2), ("c1", 8), ("c2", 2), ("c2", 4), ("c2", 8)])
def test_config_plans(cfg, P):
    c = shiro_gen.CONFIGS[cfg]
    row_ptr, col, val = shiro_gen.gen_matrix(cfg)
    part = oracle.uniform_partition(c.n, P)
    pl = sh.Plan.loopback(P, c.n, part, row_ptr, col, val, c.N, flags=sh.F_HOST_ONLY,
                          group_size=4 if P == 8 else 1)
    op = oracle.plan_flat(c.n, part, row_ptr, col)
    assert_lists_equal(pl, op, P)
    assert_stats_equal(pl, op, c.N, 4 if P == 8 else 1)
    info = pl.info()
    assert info["g_joint_rows"] < info["g_oblivious_rows"]          # north star


def test_invalid_inputs_rejected():
    n = 4
    part = np.array([0, 2, 4], np.int64)
    good = (np.array([0, 1, 2, 3, 4], np.int64), np.array([1, 0, 3, 2], np.int32),
            np.ones(4, np.float32))
    sh.Plan.loopback(2, n, part, *good, 4, flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError, match="SHIRO_E_CSR"):          # column out of range
        sh.Plan.loopback(2, n, part, good[0], np.array([1, 0, 9, 2], np.int32), good[2], 4,
                         flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError, match="SHIRO_E_CSR"):          # duplicate column
        sh.Plan.loopback(2, n, part, np.array([0, 2, 2, 3, 4], np.int64),
                         np.array([1, 1, 3, 2], np.int32), good[2], 4, flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError, match="SHIRO_E_PART"):
        sh.Plan.loopback(2, n, np.array([0, 3, 2], np.int64), *good, 4, flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError, match="SHIRO_E_ARG"):
        sh.Plan.loopback(2, n, part, *good, 0, flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError, match="SHIRO_E_ARG"):          # g must divide P
        sh.Plan.loopback(2, n, part, *good, 4, group_size=3, flags=sh.F_HOST_ONLY)


def oracle_hier_lists(msgs, P):
    """Per (stage, src, dst): B-row ids (owners ascending) then C-row ids grouped
    by final destination ascending -- the SHIRO_LIST_H*_ format."""
    out = {}
    for st in (1, 2):
        for s in range(P):
            for d in range(P):
                ms = [m for m in msgs if m.stage == st and m.src == s and m.dst == d]
                b = [m for m in ms if m.kind == "B"]
                c = [m for m in ms if m.kind in ("C", "CA")]
                b.sort(key=lambda m: m.owner if m.owner >= 0 else s)
                c.sort(key=lambda m: m.final)
                ids = [x for m in b for x in m.ids.tolist()] + [x for m in c for x in m.ids.tolist()]
                out[(st, s, d)] = np.array(ids, np.int64)
    return out


@pytest.mark.parametrize("P,g,seed", [(4, 2, 0), (8, 2, 1), (8, 4, 2), (8, 4, 3), (6, 3, 4), (8, 8, 5)])
def test_hier_lists_bit_exact(P, g, seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(80, 400))
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.01, 0.08)), symmetric=seed % 2 == 0)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 8, group_size=g, flags=sh.F_HOST_ONLY)
    op = oracle.plan_flat(n, part, row_ptr, col)
    ref = oracle_hier_lists(oracle.plan_hier(op, g), P)
    for r in range(P):
        v = pl.rank_view(r)
        for p in range(P):
            if p == r:
                continue
            for st, ks, kr in ((1, sh.LIST_H1_SEND, sh.LIST_H1_RECV), (2, sh.LIST_H2_SEND, sh.LIST_H2_RECV)):
                assert np.array_equal(v.list(p, ks), ref[(st, r, p)]), (st, r, p)
                assert np.array_equal(v.list(p, kr), ref[(st, p, r)]), (st, p, r)


@pytest.mark.parametrize("name", ["hier_col.txt", "hier_row.txt"])
def test_hier_fixture_lists(name):
    from conftest import csr_from_entries, load_golden
    meta, entries, ex = load_golden(name)
    n, P, g = meta["n"], meta["P"], meta["g"]
    row_ptr, col, val = csr_from_entries(n, entries)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 4, group_size=g, flags=sh.F_HOST_ONLY)
    info = pl.info()
    assert info["g_hier_inter_rows"] == ex["hier_inter_rows"] == 4
    assert info["g_flat_inter_rows"] == ex["flat_inter_rows"] == 8
    inter = 0
    for r in range(P):
        v = pl.rank_view(r)
        for p in range(P):
            if p != r and p // g != r // g:
                inter += v.list(p, sh.LIST_H1_SEND).size + v.list(p, sh.LIST_H2_SEND).size
    assert inter == 4                                     # 8 -> 4


def test_streamed_digests_match_full_plan_and_library():
    """oracle.plan_flat_digests (the per-rank streamed form used for c5) gives
    the same lists as plan_flat, and the library's host-only lists hash to the
    same digests (c2, P = 4)."""
    import hashlib
    from test_c5 import lib_digests
    c = shiro_gen.CONFIGS["c2"]
    rp, col, val = shiro_gen.gen_matrix("c2")
    part = oracle.uniform_partition(c.n, 4)
    dig = oracle.plan_flat_digests(c.n, part, rp, col)
    op = oracle.plan_flat(c.n, part, rp, col)
    h = lambda a: hashlib.sha256(np.asarray(a, np.int64).tobytes()).hexdigest()
    empty = np.empty(0, np.int64)
    for k, (db, dc, nb, nc) in dig.items():
        assert db == h(op.send_b.get(k, empty)) and dc == h(op.send_c.get(k, empty))
    pl = sh.Plan.loopback(4, c.n, part, rp, col, val, c.N, flags=sh.F_HOST_ONLY)
    assert lib_digests(pl, 4) == dig
