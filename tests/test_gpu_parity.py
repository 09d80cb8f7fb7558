"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north star, R11): |C - C_ref| <= max(1e-4 |C_ref|, 1e-6)
element-wise on non-negative data; exact equality on integer-mode data; plan
lists bit-exact.  Runs on one B200: P = 1 through shiro_spmm (distributed
API, no communicator) and P > 1 through the loopback ABI (all virtual ranks on
one device, device copies instead of NCCL, same planner and kernels)."""
import numpy as np
import pytest

import oracle
import shiro_gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():   # pragma: no cover - CPU boxes
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_20178_b200 as sh  # noqa: E402


def tol_ok(C, ref):
    d = np.abs(C.astype(np.float64) - ref)
    bound = np.maximum(1e-4 * np.abs(ref), 1e-6)
    bad = d > bound
    return (not bad.any()), (int(bad.sum()), float(d.max()) if d.size else 0.0)


def run_p1(n, row_ptr, col, val, B, flags=0):
    part = np.array([0, n], np.int64)
    pl = sh.Plan.distributed(0, 1, n, part, row_ptr, col, val, B.shape[1], flags=flags)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, B.shape[1]), float("nan"), device="cuda")   # must be overwritten
    pl.spmm(Bd, Cd)
    torch.cuda.synchronize()
    return Cd.cpu().numpy(), pl


def run_loopback(n, part, row_ptr, col, val, B, flags=0, group_size=1):
    P = part.size - 1
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, B.shape[1], group_size=group_size,
                          flags=flags)
    Bd = torch.from_numpy(B).cuda()
    Cd = torch.full((n, B.shape[1]), float("nan"), device="cuda")
    pl.spmm_loopback(Bd, Cd)
    torch.cuda.synchronize()
    return Cd.cpu().numpy(), pl


def hub_matrix(rng, n, hub_deg, density):
    """Random CSR plus one hub row of hub_deg nonzeros (power-law tail)."""
    m = rng.random((n, n)) < density
    m[n // 3, :] = False
    m[n // 3, rng.choice(n, size=min(hub_deg, n), replace=False)] = True
    rows, cols = np.nonzero(m)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32)


@pytest.mark.parametrize("N", [1, 3, 4, 8, 16, 32, 64, 128, 130, 256])
def test_local_spmm_widths_integer_exact(N):
    rng = np.random.default_rng(N)
    n = 3000
    row_ptr, col = hub_matrix(rng, n, 2500, 0.002)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    C, _ = run_p1(n, row_ptr, col, val, B)
    ref = oracle.spmm_ref(row_ptr, col, val, B)
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("N", [32, 64, 128])
def test_local_spmm_float_tolerance(N):
    rng = np.random.default_rng(10 + N)
    n = 5000
    row_ptr, col = hub_matrix(rng, n, 4900, 0.003)
    val = (1.0 - rng.random(col.size)).astype(np.float32)
    B = rng.random((n, N)).astype(np.float32)
    C, _ = run_p1(n, row_ptr, col, val, B)
    ok, info = tol_ok(C, oracle.spmm_ref(row_ptr, col, val, B))
    assert ok, info


def test_million_nonzero_hub_row():
    """One row with 10^6 nonzeros (split into chunk tasks) plus empty rows."""
    n, N = 1_200_000, 32
    rng = np.random.default_rng(5)
    hub_cols = np.sort(rng.choice(n, 1_000_000, replace=False)).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[8:] = hub_cols.size            # row 7 is the hub, the rest are empty
    val = rng.integers(1, 5, hub_cols.size).astype(np.float32)
    B = np.asarray(shiro_gen.gen_B(9, 0, n, N, mode=2))
    C, _ = run_p1(n, row_ptr, hub_cols, val, B)
    ref = oracle.spmm_ref(row_ptr, hub_cols, val, B, rows=np.array([7, 0, n - 1]))
    assert np.array_equal(C[[7, 0, n - 1]].astype(np.float64), ref)
    assert not C[:7].any() and not C[8:].any()


def test_empty_and_degenerate():
    n, N = 64, 32
    row_ptr = np.zeros(n + 1, np.int64)
    C, _ = run_p1(n, row_ptr, np.zeros(0, np.int32), np.zeros(0, np.float32),
                  np.ones((n, N), np.float32))
    assert not C.any()
    # empty partitions and an empty matrix through loopback
    part = np.array([0, 0, 30, 30, 64], np.int64)
    C, _ = run_loopback(n, part, row_ptr, np.zeros(0, np.int32), np.zeros(0, np.float32),
                        np.ones((n, N), np.float32))
    assert not C.any()


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("flags", [0, sh.F_SPLIT_RECV, sh.F_COVER_COLMAX, sh.F_MODE_COL,
                                   sh.F_MODE_ROW, sh.F_MODE_BLOCK, sh.F_XCHG_NCCL,
                                   sh.F_XCHG_NCCL | sh.F_SPLIT_RECV, sh.F_COVER_BALANCE])
def test_loopback_random_integer_exact(P, flags):
    rng = np.random.default_rng(P * 100 + flags)
    n, N = 2000, 64
    row_ptr, col = hub_matrix(rng, n, 1500, 0.004)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    C, _ = run_loopback(n, part, row_ptr, col, val, B, flags=flags)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_ref(row_ptr, col, val, B))


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("N", [32, 64, 128])
def test_loopback_two_phase_consumer_exact(P, N, monkeypatch):
    """The opt-in two-phase consumer CX (SHIRO_CX=1):
    per row group [local parts || remote parts], hub rows split at the local
    / remote boundary; integer data exact."""
    monkeypatch.setenv("SHIRO_CX", "1")
    monkeypatch.setenv("SHIRO_INKERNEL_WAIT", "1")
    rng = np.random.default_rng(P * 7 + N)
    n = 2500
    row_ptr, col = hub_matrix(rng, n, 2000, 0.004)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    part = oracle.uniform_partition(n, P)
    C, _ = run_loopback(n, part, row_ptr, col, val, B)
    assert np.array_equal(C.astype(np.float64), oracle.spmm_ref(row_ptr, col, val, B))


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("N", [32, 64, 128])
def test_compact_hot_buffer_exact(P, N, monkeypatch):
    """The compact hot buffer (SHIRO_HOTBUF_MB): the most
    referenced source rows of the local op are copied each step into a
    contiguous buffer read as the op's second source; integer data exact,
    one extra launch (the copy) at P = 1."""
    monkeypatch.setenv("SHIRO_HOTBUF_MB", "1")
    monkeypatch.setenv("SHIRO_HOT_MIN_MB", "0")
    rng = np.random.default_rng(P * 5 + N)
    n = 3000
    row_ptr, col = hub_matrix(rng, n, 2500, 0.004)
    val = rng.integers(1, 5, col.size).astype(np.float32)
    B = rng.integers(0, 8, (n, N)).astype(np.float32)
    ref = oracle.spmm_ref(row_ptr, col, val, B)
    if P == 1:
        pl = sh.Plan.distributed(0, 1, n, np.array([0, n], np.int64), row_ptr, col, val, N)
        for k in (1, 2, 3):            # the copy is redone every step
            Bd = torch.from_numpy(k * B).cuda()
            Cd = torch.full((n, N), float("nan"), device="cuda")
            pl.spmm(Bd, Cd)
            torch.cuda.synchronize()
            assert np.array_equal(Cd.cpu().numpy().astype(np.float64), k * ref)
            assert pl.last_launches() == 2
        return
    else:
        C, _ = run_loopback(n, oracle.uniform_partition(n, P), row_ptr, col, val, B)
    assert np.array_equal(C.astype(np.float64), ref)


@pytest.mark.parametrize("cfg,P", [("c1", 1), ("c1", 2), ("c2", 1), ("c2", 2), ("c2", 4),
                                   ("c2", 8)])
def test_config_parity(cfg, P):
    c = shiro_gen.CONFIGS[cfg]
    row_ptr, col, val = shiro_gen.gen_matrix(cfg)
    B = shiro_gen.gen_B(c.seed, 0, c.n, c.N)
    part = oracle.uniform_partition(c.n, P)
    if P == 1:
        C, pl = run_p1(c.n, row_ptr, col, val, B)
    else:
        C, pl = run_loopback(c.n, part, row_ptr, col, val, B)
        op = oracle.plan_flat(c.n, part, row_ptr, col)
        for r in range(P):
            v = pl.rank_view(r)
            for p in range(P):
                if p != r:
                    assert np.array_equal(v.list(p, sh.LIST_SEND_B),
                                          op.send_b.get((r, p), np.empty(0, np.int64)))
                    assert np.array_equal(v.list(p, sh.LIST_SEND_C),
                                          op.send_c.get((r, p), np.empty(0, np.int64)))
    ok, info = tol_ok(C, oracle.spmm_ref(row_ptr, col, val, B))
    assert ok, info
    # integer mode: exact
    _, _, vi = shiro_gen.gen_matrix(cfg, value_mode=1)
    Bi = shiro_gen.gen_B(c.seed, 0, c.n, c.N, mode=1)
    Ci = run_p1(c.n, row_ptr, col, vi, Bi)[0] if P == 1 else \
        run_loopback(c.n, part, row_ptr, col, vi, Bi)[0]
    assert np.array_equal(Ci.astype(np.float64), oracle.spmm_ref(row_ptr, col, vi, Bi))


def test_deterministic_repeat():
    c = shiro_gen.CONFIGS["c2"]
    row_ptr, col, val = shiro_gen.gen_matrix("c2")
    B = shiro_gen.gen_B(c.seed, 0, c.n, c.N)
    part = np.array([0, c.n], np.int64)
    pl = sh.Plan.distributed(0, 1, c.n, part, row_ptr, col, val, c.N)
    Bd = torch.from_numpy(B).cuda()
    C1 = torch.empty((c.n, c.N), device="cuda")
    C2 = torch.empty_like(C1)
    pl.spmm(Bd, C1)
    pl.spmm(Bd, C2)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)


def test_host_buffers_e2e():
    c = shiro_gen.CONFIGS["c1"]
    row_ptr, col, val = shiro_gen.gen_matrix("c1")
    B = shiro_gen.gen_B(c.seed, 0, c.n, c.N)
    pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), row_ptr, col, val, c.N)
    Bh = torch.from_numpy(B).pin_memory()
    Ch = torch.empty((c.n, c.N)).pin_memory()
    pl.spmm_host(Bh, Ch)
    ok, info = tol_ok(Ch.numpy(), oracle.spmm_ref(row_ptr, col, val, B))
    assert ok, info


def test_host_batch_pipelined():
    """shiro_spmm_host_batch: distinct B per item, each C exact (integer mode),
    and the pipeline must not mix items (upload i vs download i-1)."""
    c = shiro_gen.CONFIGS["c1"]
    row_ptr, col, vi = shiro_gen.gen_matrix("c1", value_mode=1)
    pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), row_ptr, col, vi, c.N)
    Bs = [torch.from_numpy(np.asarray(shiro_gen.gen_B(c.seed + i, 0, c.n, c.N, mode=1))).pin_memory()
          for i in range(5)]
    Cs = [torch.full((c.n, c.N), float("nan")).pin_memory() for _ in range(5)]
    pl.spmm_host_batch(Bs, Cs)
    for B, C in zip(Bs, Cs):
        assert np.array_equal(C.numpy().astype(np.float64),
                              oracle.spmm_ref(row_ptr, col, vi, B.numpy()))
    pl.spmm_host_batch([], [])


def test_profile_stage_times():
    c = shiro_gen.CONFIGS["c1"]
    row_ptr, col, val = shiro_gen.gen_matrix("c1")
    pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), row_ptr, col, val, c.N)
    pl.profile(True)
    Bd = torch.ones((c.n, c.N), device="cuda")
    Cd = torch.empty_like(Bd)
    pl.spmm(Bd, Cd)
    st = pl.stage_times()
    assert st["local"] > 0 and st["total"] >= st["local"]
    assert pl.last_launches() == 1
