"""Pins for the oracle's flat plan, volumes and execution simulator.

Invariants fixed by the paper: each off-diagonal nonzero is covered exactly
once (Eq. 7); mu <= min(|Rows|, |Cols|) (dominance);
joint <= col and joint <= row; bytes < the sparsity-oblivious all-gather
(north star); structural symmetry is preserved; and executing any
strategy reproduces C = A*B (P:149 four-stage execution)."""
import numpy as np
import pytest

import oracle
import shiro_gen
from conftest import random_csr


def _check_plan_invariants(n, part, row_ptr, col, plan):
    P = part.size - 1
    gi = np.repeat(np.arange(n), np.diff(row_ptr))
    po, qo = oracle.owner_of(part, gi), oracle.owner_of(part, col.astype(np.int64))
    diag = po == qo
    assert np.all(plan.tag[diag] == oracle.LOCAL)
    assert np.all(np.isin(plan.tag[~diag], [oracle.ROW, oracle.COL]))   # total & disjoint
    for p in range(P):
        for q in range(P):
            if p == q:
                continue
            sel = (po == p) & (qo == q)
            if not sel.any():
                assert (q, p) not in plan.send_b and (q, p) not in plan.send_c
                continue
            rows_u, cols_u = np.unique(gi[sel]), np.unique(col[sel])
            mu = plan.mu(q, p)
            assert mu <= min(rows_u.size, cols_u.size)                   # dominance
            assert cols_u.size <= part[q + 1] - part[q]                  # |Cols| <= K_q
            rsel = sel & (plan.tag == oracle.ROW)
            csel = sel & (plan.tag == oracle.COL)
            sc = plan.send_c.get((q, p), np.empty(0, np.int64))
            sb = plan.send_b.get((q, p), np.empty(0, np.int64))
            # lists = exactly the rows / cols used (every selected vertex is used)
            assert np.array_equal(np.unique(gi[rsel]), sc)
            assert np.array_equal(np.unique(col[csel]).astype(np.int64), sb)
            assert np.all(np.diff(sc) > 0) and np.all(np.diff(sb) > 0)
            assert np.all((part[p] <= sc) & (sc < part[p + 1]))
            assert np.all((part[q] <= sb) & (sb < part[q + 1]))


@pytest.mark.parametrize("seed", range(54))
def test_random_plan_invariants_and_dominance(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(30, 400)) if seed % 9 else 1000
    P = [2, 4, 8][seed % 3]
    sym = seed % 2 == 0
    row_ptr, col, val = random_csr(rng, n, float(rng.uniform(0.002, 0.05)), symmetric=sym)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col)
    _check_plan_invariants(n, part, row_ptr, col, plan)
    v = oracle.volumes(plan, N=32)
    assert v["joint_rows"] <= v["col_rows"] and v["joint_rows"] <= v["row_rows"]
    assert v["col_rows"] <= v["block_rows"] and v["block_rows"] <= v["oblivious_rows"]
    assert v["joint_bytes"] == v["joint_rows"] * 32 * 4
    if sym:
        pr = v["pair_rows"]
        assert np.array_equal(pr, pr.T)
    # the col-max rule moves work but not bytes (R1)
    plan_c = oracle.plan_flat(n, part, row_ptr, col, rule="colmax")
    _check_plan_invariants(n, part, row_ptr, col, plan_c)
    assert oracle.volumes(plan_c, 32)["joint_rows"] == v["joint_rows"]
    # single strategies (Eqs. 2-3)
    pc = oracle.plan_flat(n, part, row_ptr, col, mode="col")
    pr_ = oracle.plan_flat(n, part, row_ptr, col, mode="row")
    assert oracle.volumes(pc, 32)["joint_rows"] == v["col_rows"]
    assert oracle.volumes(pr_, 32)["joint_rows"] == v["row_rows"]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("mode,rule", [("joint", "rowmax"), ("joint", "colmax"),
                                       ("col", "rowmax"), ("row", "rowmax")])
def test_exec_flat_reproduces_product(P, mode, rule):
    rng = np.random.default_rng(P * 10 + len(mode))
    n, N = 96, 5
    row_ptr, col, val = random_csr(rng, n, 0.06)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    plan = oracle.plan_flat(n, part, row_ptr, col, mode=mode, rule=rule)
    C = oracle.exec_flat(plan, row_ptr, col, val, B)
    assert np.array_equal(C, oracle.spmm_ref(row_ptr, col, val, B))     # integer: exact
    Bf = rng.random((n, N)).astype(np.float32)
    valf = rng.random(val.size).astype(np.float32)
    Cf = oracle.exec_flat(plan, row_ptr, col, valf, Bf)
    ref = oracle.spmm_ref(row_ptr, col, valf, Bf)
    assert np.allclose(Cf, ref, rtol=1e-12, atol=1e-300)


def test_exec_detects_missing_b_row():
    rng = np.random.default_rng(5)
    n = 40
    row_ptr, col, val = random_csr(rng, n, 0.1)
    part = oracle.uniform_partition(n, 2)
    plan = oracle.plan_flat(n, part, row_ptr, col, mode="col")
    key = next(iter(plan.send_b))
    plan.send_b[key] = plan.send_b[key][1:]
    with pytest.raises(RuntimeError, match="coverage"):
        oracle.exec_flat(plan, row_ptr, col, val, np.ones((n, 2), np.float32))


def test_c1_config_bytes_below_oblivious():
    cfg = shiro_gen.CONFIGS["c1"]
    row_ptr, col, val = shiro_gen.gen_matrix("c1")
    assert row_ptr[-1] == cfg.nnz
    for P in (2, 4, 8):
        part = oracle.uniform_partition(cfg.n, P)
        plan = oracle.plan_flat(cfg.n, part, row_ptr, col)
        v = oracle.volumes(plan, cfg.N)
        assert v["joint_bytes"] < v["oblivious_bytes"]
        assert v["joint_rows"] <= min(v["col_rows"], v["row_rows"])


def test_block_mode_is_eq1():
    """Sparsity-oblivious block strategy (Eq. 1): per non-empty
    block q sends all K_q rows; the executed product is still exact."""
    rng = np.random.default_rng(77)
    n, P = 120, 4
    row_ptr, col, val = random_csr(rng, n, 0.03)
    part = oracle.uniform_partition(n, P)
    pb = oracle.plan_flat(n, part, row_ptr, col, mode="block")
    v = oracle.volumes(pb, 8)
    assert v["joint_rows"] == v["block_rows"]
    B = rng.integers(0, 8, (n, 3)).astype(np.float32)
    assert np.array_equal(oracle.exec_flat(pb, row_ptr, col, val, B),
                          oracle.spmm_ref(row_ptr, col, val, B))
