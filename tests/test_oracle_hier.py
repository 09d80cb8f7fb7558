"""Pins for the oracle's hierarchical plan (Algorithm 1).

Fixed by the paper: the 8 -> 4 inter-group reductions of both worked examples
(L517, L519, tests/golden/hier_*.txt); degenerate topologies (g = 1 is flat,
g = P has no inter-group traffic); uniqueness of every (owner, B
row, destination group) and (source group, C row, destination) crossing
(S:373-374); inter-group bytes never above the flat plan's (L782);
stage/tier purity (Alg. 1); and execution reproduces C = A*B."""
import numpy as np
import pytest

import oracle
from conftest import csr_from_entries, load_golden, random_csr


@pytest.mark.parametrize("name", ["hier_col.txt", "hier_row.txt"])
def test_paper_8_to_4_fixtures(name):
    meta, entries, ex = load_golden(name)
    n, P, g = meta["n"], meta["P"], meta["g"]
    row_ptr, col, val = csr_from_entries(n, entries)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col)
    msgs = oracle.plan_hier(plan, g)
    tt = oracle.tier_traffic(msgs, N=1, sz=1)
    assert oracle.flat_inter_rows(plan, g) == ex["flat_inter_rows"] == 8
    assert tt["inter_rows"] == ex["hier_inter_rows"] == 4
    assert tt["intra_rows"] == ex["hier_intra_rows"]
    B = np.arange(n * 3, dtype=np.float32).reshape(n, 3) % 7
    C = oracle.exec_hier(plan, msgs, g, row_ptr, col, val, B)
    assert np.array_equal(C, oracle.spmm_ref(row_ptr, col, val, B))


def _check_schedule(plan, msgs, g):
    grp = lambda r: r // g
    for m in msgs:
        assert m.src != m.dst
        inter = grp(m.src) != grp(m.dst)
        assert (m.tier == "inter") == inter                              # tier purity
        if m.stage == 1 and inter:
            assert m.kind == "B"                                         # I.1 column fetch
        if m.stage == 2 and inter:
            assert m.kind == "CA"                                        # II.2 row transmission
        if m.stage == 2 and not inter:
            assert m.kind == "B"                                         # II.2 column distribution
    seen_b, seen_c = set(), set()
    for m in msgs:
        if m.tier != "inter":
            continue
        for r in m.ids.tolist():
            if m.kind == "B":
                key = (m.src, r, grp(m.dst))
                assert key not in seen_b; seen_b.add(key)
            else:
                key = (grp(m.src), r, m.dst)
                assert key not in seen_c; seen_c.add(key)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("P,g", [(4, 2), (8, 2), (8, 4)])
def test_random_hier(seed, P, g):
    rng = np.random.default_rng(seed + 100 * P + g)
    n, N = int(rng.integers(40, 160)), 3
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.02, 0.12)), symmetric=seed % 2 == 0)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col)
    msgs = oracle.plan_hier(plan, g)
    _check_schedule(plan, msgs, g)
    tt = oracle.tier_traffic(msgs, N=1, sz=1)
    assert tt["inter_rows"] <= oracle.flat_inter_rows(plan, g)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    C = oracle.exec_hier(plan, msgs, g, row_ptr, col, val, B)
    assert np.array_equal(C, oracle.spmm_ref(row_ptr, col, val, B))


def test_degenerate_groups():
    rng = np.random.default_rng(7)
    n, P = 120, 8
    row_ptr, col, val = random_csr(rng, n, 0.05)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col)
    flat_total = sum(plan.mu(q, p) for (q, p) in plan.n_cols)
    m1 = oracle.plan_hier(plan, 1)                                       # g = 1: flat
    t1 = oracle.tier_traffic(m1, 1, 1)
    assert t1["intra_rows"] == 0 and t1["inter_rows"] == flat_total
    mP = oracle.plan_hier(plan, P)                                       # g = P: one group
    tP = oracle.tier_traffic(mP, 1, 1)
    assert tP["inter_rows"] == 0 and tP["intra_rows"] == flat_total
    B = rng.integers(0, 8, (n, 2)).astype(np.float32)
    ref = oracle.spmm_ref(row_ptr, col, val, B)
    for msgs, g in ((m1, 1), (mP, P)):
        assert np.array_equal(oracle.exec_hier(plan, msgs, g, row_ptr, col, val, B), ref)
