"""Weighted covers (Eqs. 4-8, weighted
network L372-375): the library's weighted plans (Dinic in cover.cpp, host
only, loopback) against the oracle's (Dinic in oracle_core.c, brute-force
pinned in test_oracle_cover.py), plus closed forms that fix the weighted
optimum without either implementation:
  * w_col >> w_row (B rows expensive): the cover is all rows -> the row-based
    plan (Eq. 3), every off-diagonal nonzero ROW;
  * w_row >> w_col: all columns -> the column-based plan (Eq. 2);
  * uniform weights: identical to the unit-weight (Hopcroft-Karp) plan."""
import numpy as np
import pytest

import oracle
import paper_2512_20178_b200 as sh
from conftest import random_csr
from test_planner_parity import assert_lists_equal

BIG = 10 ** 6


def _plan_lib(n, part, row_ptr, col, val, w_row, w_col, flags=0):
    return sh.Plan.loopback(part.size - 1, n, part, row_ptr, col, val, 8,
                            flags=flags | sh.F_HOST_ONLY, w_row=w_row, w_col=w_col)


@pytest.mark.parametrize("seed", range(24))
def test_weighted_lists_match_oracle(seed):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(8, 200))
    P = [2, 3, 4][seed % 3]
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.01, 0.2)), symmetric=seed % 2 == 0)
    part = oracle.uniform_partition(n, P)
    w_row = rng.integers(1, 9, n).astype(np.int64)
    w_col = rng.integers(1, 9, n).astype(np.int64)
    rule = "colmax" if seed % 4 == 3 else "rowmax"
    op = oracle.plan_flat(n, part, row_ptr, col, rule=rule, w_row=w_row, w_col=w_col)
    pl = _plan_lib(n, part, row_ptr, col, val, w_row, w_col,
                   sh.F_COVER_COLMAX if rule == "colmax" else 0)
    assert_lists_equal(pl, op, P)
    # the weighted optimum never costs more than either one-sided plan
    cost = lambda p: sum(int(w_row[p.send_c[k]].sum()) for k in p.send_c) + \
        sum(int(w_col[p.send_b[k]].sum()) for k in p.send_b)
    assert cost(op) <= cost(oracle.plan_flat(n, part, row_ptr, col, mode="col"))
    assert cost(op) <= cost(oracle.plan_flat(n, part, row_ptr, col, mode="row"))


@pytest.mark.parametrize("expensive", ["col", "row"])
def test_weighted_extremes_are_one_sided_plans(expensive):
    rng = np.random.default_rng(11)
    n, P = 120, 4
    row_ptr, col, val = random_csr(rng, n, 0.05)
    part = oracle.uniform_partition(n, P)
    w_row = np.full(n, BIG if expensive == "row" else 1, np.int64)
    w_col = np.full(n, BIG if expensive == "col" else 1, np.int64)
    one_sided = oracle.plan_flat(n, part, row_ptr, col, mode="row" if expensive == "col" else "col")
    op = oracle.plan_flat(n, part, row_ptr, col, w_row=w_row, w_col=w_col)
    assert_lists_equal(_plan_lib(n, part, row_ptr, col, val, w_row, w_col), one_sided, P)
    assert_lists_equal(_plan_lib(n, part, row_ptr, col, val, w_row, w_col), op, P)


def test_uniform_weights_equal_unit_plan():
    rng = np.random.default_rng(5)
    n, P = 150, 3
    row_ptr, col, val = random_csr(rng, n, 0.04, symmetric=True)
    part = oracle.uniform_partition(n, P)
    ones = np.ones(n, np.int64)
    assert_lists_equal(_plan_lib(n, part, row_ptr, col, val, ones * 3, ones * 3),
                       oracle.plan_flat(n, part, row_ptr, col), P)


def test_weighted_rejects_bad_weights():
    rng = np.random.default_rng(1)
    n, P = 40, 2
    row_ptr, col, val = random_csr(rng, n, 0.2)
    part = oracle.uniform_partition(n, P)
    w = np.ones(n, np.int64)
    w[:] = 0
    with pytest.raises(sh.ShiroError):
        _plan_lib(n, part, row_ptr, col, val, w, np.ones(n, np.int64))


def test_refresh_needs_device_state():
    rng = np.random.default_rng(2)
    n = 50
    row_ptr, col, val = random_csr(rng, n, 0.1)
    part = oracle.uniform_partition(n, 2)
    pl = sh.Plan.loopback(2, n, part, row_ptr, col, val, 8, flags=sh.F_HOST_ONLY)
    with pytest.raises(sh.ShiroError):
        pl.update_values(val, stream=0)
