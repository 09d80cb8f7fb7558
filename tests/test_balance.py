"""SHIRO_F_COVER_BALANCE (R18, not from the paper): a block whose
all-rows cover is within max(1, mu/1000) rows of the minimum cover mu is
covered by all its rows, so the column owner computes it.

Pins (CPU): a hand-built complete bipartite block K_{5,4} (mu = 4 columns,
all rows = 5 = mu + 1 -> rows); exec-sim of balanced plans reproduces the
product exactly (every nonzero covered once); the byte increase is bounded by
the slack per block; on a symmetric dense-ish matrix with an odd n (the c3
situation) the balanced plan splits the off-diagonal compute evenly where
the minimum cover puts all of it on one rank; the library's lists equal the
oracle's bit for bit."""
import numpy as np
import pytest

import oracle
import paper_2512_20178_b200 as sh
from conftest import random_csr


def _k54():
    # rows 0..4 (rank 0) x cols 5..8 (rank 1), complete; rank 1 rows empty
    n = 9
    part = np.array([0, 5, 9], np.int64)
    rows = np.repeat(np.arange(5), 4)
    cols = np.tile(np.arange(5, 9), 5)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return n, part, row_ptr, cols.astype(np.int32)


def test_k54_block_goes_to_rows():
    n, part, row_ptr, col = _k54()
    base = oracle.plan_flat(n, part, row_ptr, col)
    assert np.array_equal(base.send_b[(1, 0)], np.arange(5, 9))      # min cover: 4 columns
    assert (1, 0) not in base.send_c
    bal = oracle.plan_flat(n, part, row_ptr, col, balance=True)
    assert np.array_equal(bal.send_c[(1, 0)], np.arange(5))            # 5 rows = mu + 1
    assert (1, 0) not in bal.send_b
    assert oracle.balance_slack(4) == 1 and oracle.balance_slack(2500) == 2


def _computed_nnz(plan, row_ptr, col, part):
    """Off-diagonal nonzeros computed per rank: ROW -> column owner, COL -> row owner."""
    P = part.size - 1
    gi = np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))
    po, qo = oracle.owner_of(part, gi), oracle.owner_of(part, col)
    work = np.zeros(P, np.int64)
    for (q, p), rows in plan.send_c.items():
        m = (po == p) & (qo == q)
        is_row = np.isin(gi[m], rows)
        work[q] += int(is_row.sum())
        work[p] += int((~is_row).sum())
    for (q, p), cols in plan.send_b.items():
        if (q, p) in plan.send_c:
            continue
        work[p] += int(((po == p) & (qo == q)).sum())
    return work


def test_symmetric_dense_odd_n_balances_compute():
    rng = np.random.default_rng(7)
    n = 101                                   # odd: blocks of 51 and 50 rows
    row_ptr, col, val = random_csr(rng, n, 0.6, symmetric=True)
    part = oracle.uniform_partition(n, 2)
    base = oracle.plan_flat(n, part, row_ptr, col)
    bal = oracle.plan_flat(n, part, row_ptr, col, balance=True)
    wb, wl = _computed_nnz(base, row_ptr, col, part), _computed_nnz(bal, row_ptr, col, part)
    assert wb.min() == 0                      # minimum cover: one rank computes both blocks
    assert abs(int(wl[0]) - int(wl[1])) <= 0.1 * wl.sum()
    vb, vl = oracle.volumes(base, 8), oracle.volumes(bal, 8)
    assert vb["joint_rows"] <= vl["joint_rows"] <= vb["joint_rows"] + 2


@pytest.mark.parametrize("seed", range(12))
def test_balanced_plans_exact_and_bounded(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(20, 200))
    P = [2, 3, 4][seed % 3]
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.01, 0.7)), symmetric=seed % 2 == 0)
    part = oracle.uniform_partition(n, P)
    base = oracle.plan_flat(n, part, row_ptr, col)
    bal = oracle.plan_flat(n, part, row_ptr, col, balance=True)
    # each block either keeps its minimum cover or switches to all of its rows
    slack = 0
    for key in set(base.n_rows) | set(bal.n_rows):
        mu = base.send_b.get(key, np.empty(0)).size + base.send_c.get(key, np.empty(0)).size
        got = bal.send_b.get(key, np.empty(0)).size + bal.send_c.get(key, np.empty(0)).size
        if got != mu or key in bal.send_b and not np.array_equal(bal.send_b[key], base.send_b.get(key)):
            assert key not in bal.send_b and bal.send_c[key].size == base.n_rows[key]
            assert got <= mu + oracle.balance_slack(mu)
            slack += got - mu
    assert oracle.volumes(bal, 4)["joint_rows"] == oracle.volumes(base, 4)["joint_rows"] + slack
    B = rng.integers(0, 8, (n, 8)).astype(np.float32)
    C = oracle.exec_flat(bal, row_ptr, col, val, B)
    assert np.array_equal(C, oracle.spmm_ref(row_ptr, col, val, B))


@pytest.mark.parametrize("seed", range(10))
def test_library_balanced_lists_bit_exact(seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(30, 250))
    P = [2, 3, 4, 8][seed % 4]
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.02, 0.6)), symmetric=seed % 2 == 0)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 16,
                          flags=sh.F_COVER_BALANCE | sh.F_HOST_ONLY)
    op = oracle.plan_flat(n, part, row_ptr, col, balance=True)
    empty = np.empty(0, np.int64)
    for r in range(P):
        v = pl.rank_view(r)
        for p in range(P):
            if p != r:
                assert np.array_equal(v.list(p, sh.LIST_SEND_B), op.send_b.get((r, p), empty))
                assert np.array_equal(v.list(p, sh.LIST_SEND_C), op.send_c.get((r, p), empty))
    assert pl.info()["g_joint_rows"] == oracle.volumes(op, 16)["joint_rows"]
