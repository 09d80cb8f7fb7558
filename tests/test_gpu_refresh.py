"""GPU: value refresh for a fixed pattern (PAPER.md L300:
the plan is reused "across multiple SpMM operations with the same sparsity
pattern") and weighted covers executed end to end (N2; L315-337).

A plan built with values v1 and refreshed to v2 must compute A(v2)*B exactly
(integer mode) -- for the fused, split, NCCL-staged, transposed and
hierarchical schedules -- and a weighted plan must compute the same product as
any other plan (the cover only moves the work)."""
import numpy as np
import pytest

import oracle
import shiro_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():   # pragma: no cover - CPU boxes
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_20178_b200 as sh  # noqa: E402
from test_gpu_parity import hub_matrix  # noqa: E402


def _transpose(n, row_ptr, col, val):
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    order = np.lexsort((rows, col))
    t_rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(col, minlength=n), out=t_rp[1:])
    return t_rp, rows[order].astype(np.int32), val[order]


@pytest.mark.parametrize("P,g,flags", [(1, 1, 0), (2, 1, 0), (4, 1, 0), (3, 1, sh.F_SPLIT_RECV),
                                       (4, 1, sh.F_XCHG_NCCL), (4, 1, sh.F_COVER_COLMAX),
                                       (4, 2, 0), (3, 1, sh.F_TRANSPOSE),
                                       (4, 2, sh.F_TRANSPOSE)])
def test_loopback_refresh_exact(P, g, flags):
    rng = np.random.default_rng(100 * P + g + flags)
    n, N = 1500, 64
    row_ptr, col = hub_matrix(rng, n, 1200, 0.004)
    v1 = rng.integers(1, 5, col.size).astype(np.float32)
    v2 = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, v1, N, group_size=g, flags=flags)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, N), float("nan"), device="cuda")
    ref = lambda v: (oracle.spmm_ref(*_transpose(n, row_ptr, col, v), B)
                     if flags & sh.F_TRANSPOSE else oracle.spmm_ref(row_ptr, col, v, B))
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    assert np.array_equal(Cd.cpu().numpy().astype(np.float64), ref(v1))
    pl.update_values(v2)
    Cd.fill_(float("nan"))
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    assert np.array_equal(Cd.cpu().numpy().astype(np.float64), ref(v2))
    assert pl.info()["refresh_seconds"] > 0


def test_distributed_P1_refresh_and_graph_replay():
    """P = 1 through shiro_spmm on a capturable stream: the refresh must be
    seen by the replayed CUDA graph (values are rewritten in place)."""
    c = shiro_gen.CONFIGS["c2"]
    rp, col, _ = shiro_gen.gen_matrix("c2")
    v1 = shiro_gen.gen_values("c2", rp, col, 1)
    v2 = np.where(v1 > 2, v1 - 1, v1 + 1).astype(np.float32)
    Bi = shiro_gen.gen_B(c.seed, 0, c.n, c.N, mode=1)
    pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), rp, col, v1, c.N)
    s = torch.cuda.Stream()
    Bd = torch.from_numpy(Bi).cuda()
    Cd = torch.empty((c.n, c.N), device="cuda")
    for i, v in enumerate((v1, v2, v1)):
        if i > 0:
            pl.update_values(v, stream=s)
        pl.spmm(Bd, Cd, s)
        pl.spmm(Bd, Cd, s)       # second call replays the graph
        s.synchronize()
        assert np.array_equal(Cd.cpu().numpy().astype(np.float64),
                              oracle.spmm_ref(rp, col, v, Bi))


@pytest.mark.parametrize("P", [2, 4])
def test_weighted_plan_product_exact(P):
    rng = np.random.default_rng(P)
    n, N = 2000, 32
    row_ptr, col = hub_matrix(rng, n, 1500, 0.003)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    w_row = rng.integers(1, 6, n).astype(np.int64)
    w_col = rng.integers(1, 6, n).astype(np.int64)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, N, w_row=w_row, w_col=w_col)
    op = oracle.plan_flat(n, part, row_ptr, col, w_row=w_row, w_col=w_col)
    from test_planner_parity import assert_lists_equal
    assert_lists_equal(pl, op, P)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, N), float("nan"), device="cuda")
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    assert np.array_equal(Cd.cpu().numpy().astype(np.float64), oracle.spmm_ref(row_ptr, col, val, B))
