"""GPU parity at FULL size on the large configs (north star: "bit-exact plans
and C within 1e-4 relative error of the oracle on all five configs"; SURVEY
8(c) step 9; PAPER.md L138 is the definition C = A*B the oracle computes).

c3 (Reddit-shaped, 114.6 M nonzeros) and c4 (ogbn-products-shaped, 61.9 M)
at P = 1 through shiro_spmm reach the kernel instantiations the benchmark
runs: 256-nonzero work units, hub-row chunk tasks, source rows far larger
than L2 (no L2 policy) and, with SHIRO_HOT_MB, the hot/cold L2 marks.  P = 4
and P = 8 run the multi-rank planner, fused producer and per-source consumer
through the loopback ABI; their lists must equal the oracle's bit-exactly.
Every element is compared: non-negative data within the R11 tolerance,
integer-mode data exactly (R11).  c5 (1.07 B nonzeros) is covered
by tests/test_c5.py (list digests + sampled rows)."""
import os

import numpy as np
import pytest

import oracle
import shiro_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():   # pragma: no cover - CPU boxes
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_20178_b200 as sh  # noqa: E402
from test_gpu_parity import run_loopback, run_p1, tol_ok  # noqa: E402
from test_planner_parity import assert_lists_equal  # noqa: E402

_CACHE = {}


def config(name):
    """(cfg, row_ptr, col, val, val_int, B, B_int), generated once per session."""
    if name not in _CACHE:
        c = shiro_gen.CONFIGS[name]
        rp, col, val = shiro_gen.gen_matrix(name, cache_dir=os.environ.get("SHIRO_GEN_CACHE"))
        vi = shiro_gen.gen_values(name, rp, col, 1)
        B = shiro_gen.gen_B(c.seed, 0, c.n, c.N)
        Bi = shiro_gen.gen_B(c.seed, 0, c.n, c.N, mode=1)
        _CACHE[name] = (c, rp, col, val, vi, B, Bi)
    return _CACHE[name]


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_config_P1(name):
    c, rp, col, val, vi, B, Bi = config(name)
    C, pl = run_p1(c.n, rp, col, val, B)
    info = pl.info()
    assert info["nnz_local"] == rp[-1]
    ok, bad = tol_ok(C, oracle.spmm_ref(rp, col, val, B))
    assert ok, bad
    del C
    Ci, _ = run_p1(c.n, rp, col, vi, Bi)
    assert np.array_equal(Ci.astype(np.float64), oracle.spmm_ref(rp, col, vi, Bi))


def test_c4_P1_hot_cold_l2_marks(monkeypatch):
    """The hot/cold L2 policy variant (kHotBit marks) on c4, integer exact."""
    monkeypatch.setenv("SHIRO_HOT_MB", "64")
    c, rp, col, val, vi, B, Bi = config("c4")
    Ci, _ = run_p1(c.n, rp, col, vi, Bi)
    assert np.array_equal(Ci.astype(np.float64), oracle.spmm_ref(rp, col, vi, Bi))


@pytest.mark.parametrize("name,P", [("c3", 4), ("c3", 8), ("c4", 4), ("c4", 8)])
def test_full_config_loopback(name, P):
    c, rp, col, val, vi, B, Bi = config(name)
    part = oracle.uniform_partition(c.n, P)
    op = oracle.plan_flat(c.n, part, rp, col)
    C, pl = run_loopback(c.n, part, rp, col, val, B)
    assert_lists_equal(pl, op, P)
    ok, bad = tol_ok(C, oracle.spmm_ref(rp, col, val, B))
    assert ok, bad
    del C, pl
    Ci, _ = run_loopback(c.n, part, rp, col, vi, Bi)
    assert np.array_equal(Ci.astype(np.float64), oracle.spmm_ref(rp, col, vi, Bi))
