"""Pins for the oracle's minimum vertex cover.

Checked against: the worked examples of Fig. 1 and Fig. 4 (tests/golden), the
sparsity patterns of Fig. 5, closed forms (K_{m,k}, single edge), exhaustive
brute force on tiny blocks (minimum weight AND the canonical cut = union of
row sets / intersection of column sets over all minimum covers), and König's
theorem via an independent matching algorithm (Kuhn)."""
import numpy as np
import pytest

import oracle
from conftest import csr_from_entries, load_golden


def _block_pair_stats(name):
    meta, entries, expect = load_golden(name)
    n, P = meta["n"], meta["P"]
    row_ptr, col, val = csr_from_entries(n, entries)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col)
    return plan, expect, (n, part, row_ptr, col)


def test_fig1_worked_example():
    plan, ex, (n, part, row_ptr, col) = _block_pair_stats("fig1.txt")
    assert part.tolist() == [0, 4, 8]
    v = oracle.volumes(plan, N=1, sz=1)
    assert v["col_rows"] == ex["col_rows"] == 3          # L101
    assert v["row_rows"] == ex["row_rows"] == 3          # L111
    assert v["joint_rows"] == ex["joint_rows"] == 2      # L120, L236
    assert v["block_rows"] == ex["block_rows"] == 4      # Eq. 1 with K = 4
    assert plan.send_c[(1, 0)].tolist() == [ex["cover_rows"]]   # C row 0 (L306)
    assert plan.send_b[(1, 0)].tolist() == [ex["cover_cols"]]   # B row 6 (L306)
    assert abs(v["red_col"] - (1 - 2 / 3)) < 1e-15 and abs(v["red_row"] - (1 - 2 / 3)) < 1e-15
    # col-based and row-based plans reproduce Fig. 1(b) and 1(c)
    pc = oracle.plan_flat(n, part, row_ptr, col, mode="col")
    pr = oracle.plan_flat(n, part, row_ptr, col, mode="row")
    assert pc.send_b[(1, 0)].tolist() == [5, 6, 7] and (1, 0) not in pc.send_c
    assert pr.send_c[(1, 0)].tolist() == [0, 1, 2] and (1, 0) not in pr.send_b
    # assignment of SPEC L224: b,d -> row-based; f,h -> col-based; c doubly covered -> ROW
    tags = dict(zip(zip(np.repeat(np.arange(n), np.diff(row_ptr)).tolist(), col.tolist()),
                    plan.tag.tolist()))
    assert tags[(0, 5)] == oracle.ROW and tags[(0, 7)] == oracle.ROW
    assert tags[(0, 6)] == oracle.ROW
    assert tags[(1, 6)] == oracle.COL and tags[(2, 6)] == oracle.COL
    assert tags[(0, 0)] == oracle.LOCAL


def test_fig4_worked_example():
    plan, ex, _ = _block_pair_stats("fig4.txt")
    assert plan.mu(1, 0) == ex["joint_rows"] == 2
    assert plan.send_c[(1, 0)].tolist() == [ex["cover_rows"]]
    assert plan.send_b[(1, 0)].tolist() == [ex["cover_cols"]]


def _pattern_edges(name, s, h):
    if name == "pattern3":
        return [(i, i) for i in range(s)]
    if name == "pattern4":
        return sorted({(0, j) for j in range(s)} | {(i, 0) for i in range(s)})
    if name == "pattern1":
        return [(i, j) for i in range(h) for j in range(s)]
    if name == "pattern2":
        return [(i, j) for i in range(s) for j in range(h)]
    raise ValueError(name)


def test_fig5_patterns():
    with open(__import__("conftest").GOLDEN + "/patterns.txt") as f:
        lines = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    assert len(lines) >= 4
    for name, s, h, mu, red_col, red_row in lines:
        s, h, mu = int(s), int(h), int(mu)
        edges = _pattern_edges(name, s, h)
        er, ec = [e[0] for e in edges], [e[1] for e in edges]
        nr, nc = max(er) + 1, max(ec) + 1
        sr, sc, flow = oracle.min_cover_local(nr, nc, er, ec)
        assert flow == mu == sr.sum() + sc.sum(), name
        assert abs((1 - mu / nc) - float(red_col)) < 1e-12, name       # Eq. 11
        assert abs((1 - mu / nr) - float(red_row)) < 1e-12, name
        if name == "pattern4":
            assert sr.tolist() == [True] + [False] * (s - 1)            # row 0 + col 0
            assert sc.tolist() == [True] + [False] * (s - 1)
        if name == "pattern3":
            assert sr.all() and not sc.any()                            # row-max tie rule


@pytest.mark.parametrize("m,k", [(1, 1), (1, 5), (3, 3), (4, 2), (2, 7), (6, 6)])
def test_complete_bipartite_closed_form(m, k):
    er = [i for i in range(m) for _ in range(k)]
    ec = [j for _ in range(m) for j in range(k)]
    sr, sc, flow = oracle.min_cover_local(m, k, er, ec)
    assert flow == min(m, k)
    # canonical row-max: rows whenever rows are a minimum cover
    if m <= k:
        assert sr.all() and not sc.any()
    else:
        assert sc.all() and not sr.any()
    sr2, sc2, _ = oracle.min_cover_local(m, k, er, ec, rule="colmax")
    if k <= m:
        assert sc2.all() and not sr2.any()
    else:
        assert sr2.all() and not sc2.any()


def test_single_edge_and_weights():
    sr, sc, f = oracle.min_cover_local(1, 1, [0], [0])
    assert f == 1 and sr.tolist() == [True] and sc.tolist() == [False]
    sr, sc, f = oracle.min_cover_local(1, 1, [0], [0], rule="colmax")
    assert f == 1 and sr.tolist() == [False] and sc.tolist() == [True]
    # cheaper side forced
    sr, sc, f = oracle.min_cover_local(1, 1, [0], [0], w_row=[1], w_col=[5])
    assert f == 1 and sr.tolist() == [True]
    sr, sc, f = oracle.min_cover_local(1, 1, [0], [0], w_row=[5], w_col=[1], rule="rowmax")
    assert f == 1 and sc.tolist() == [True]


def _random_instance(rng, max_side):
    nr = int(rng.integers(1, max_side + 1))
    nc = int(rng.integers(1, max_side + 1))
    dens = rng.uniform(0.1, 0.8)
    edges = [(i, j) for i in range(nr) for j in range(nc) if rng.random() < dens]
    if not edges:
        edges = [(int(rng.integers(nr)), int(rng.integers(nc)))]
    # keep only vertices that carry an edge (Rows/Cols are index sets of nonzeros)
    rs = sorted({e[0] for e in edges})
    cs = sorted({e[1] for e in edges})
    rmap, cmap = {r: t for t, r in enumerate(rs)}, {c: t for t, c in enumerate(cs)}
    return len(rs), len(cs), [(rmap[i], cmap[j]) for i, j in edges]


def test_brute_force_optimality_konig_and_canonical_cut():
    """>= 500 random instances: Dinic's cover weight equals the
    exhaustive minimum; flow = cover weight = maximum matching (König); the
    row-max / col-max cuts equal (union rows, intersection cols) /
    (intersection rows, union cols) over all minimum covers."""
    rng = np.random.default_rng(1234)
    for t in range(520):
        nr, nc, edges = _random_instance(rng, 8 if t < 400 else 10)
        er, ec = [e[0] for e in edges], [e[1] for e in edges]
        weighted = t % 3 == 2
        wr = rng.integers(1, 6, nr).tolist() if weighted else None
        wc = rng.integers(1, 6, nc).tolist() if weighted else None
        best, covers = oracle.brute_force_cover(nr, nc, edges, wr, wc)
        for rule in ("rowmax", "colmax"):
            sr, sc, flow = oracle.min_cover_local(nr, nc, er, ec, wr, wc, rule=rule)
            w = (np.array(wr) if wr else np.ones(nr, int))[sr].sum() + \
                (np.array(wc) if wc else np.ones(nc, int))[sc].sum()
            assert flow == best == w
            got = (frozenset(np.nonzero(sr)[0].tolist()), frozenset(np.nonzero(sc)[0].tolist()))
            assert got in covers
            if rule == "rowmax":
                expect = (frozenset().union(*[c[0] for c in covers]),
                          frozenset.intersection(*[c[1] for c in covers]))
            else:
                expect = (frozenset.intersection(*[c[0] for c in covers]),
                          frozenset().union(*[c[1] for c in covers]))
            assert got == expect
        if not weighted:
            assert oracle.max_matching_kuhn(nr, nc, edges) == best


def test_konig_on_larger_blocks():
    rng = np.random.default_rng(99)
    for _ in range(30):
        nr, nc = int(rng.integers(20, 120)), int(rng.integers(20, 120))
        m = rng.random((nr, nc)) < rng.uniform(0.01, 0.1)
        er, ec = np.nonzero(m)
        if er.size == 0:
            continue
        sr, sc, flow = oracle.min_cover_local(nr, nc, er, ec)
        assert flow == oracle.max_matching_kuhn(nr, nc, list(zip(er.tolist(), ec.tolist())))
        assert np.all(sr[er] | sc[ec])                                  # Eq. 7
        assert sr.sum() + sc.sum() == flow


def test_uniform_partition_larger_blocks_first():
    """S:101 / S:104-106: sizes ceil/floor(n/P), the larger blocks first
    (10 rows over 4 ranks: 3, 3, 2, 2)."""
    assert oracle.uniform_partition(10, 4).tolist() == [0, 3, 6, 8, 10]
    assert oracle.uniform_partition(3, 5).tolist() == [0, 1, 2, 3, 3, 3]   # empty blocks
    assert oracle.uniform_partition(8, 2).tolist() == [0, 4, 8]


def test_fig1_setup_bytes():
    """Fig. 1: the joint cover sends C row 0, whose row-based
    nonzeros b, c, d (3 entries) are shipped once at plan time:
    3 x (4 B column + 4 B value) = 24 B (R14)."""
    plan, _, _ = _block_pair_stats("fig1.txt")
    assert plan.nnz_row[(1, 0)] == 3
    assert oracle.volumes(plan, N=1)["setup_bytes"] == 24
