"""GPU: the multi-rank distributed path (shiro_plan / shiro_spmm with the fused
NVLink exchange) in several OS processes sharing cuda:0.

Each process is one rank: the plan-time exchange runs over gloo (caller
transport, no NCCL communicator), the per-step exchange is the fused one --
CUDA-IPC peer stores into the other processes' receive buffers plus epoch
flags, the producer on a high-priority stream concurrent with the local SpMM,
per-source waits in the consumer -- exactly the code the multi-GPU runs use,
here on one device.  Several steps with different B exercise the
double-buffered receive buffers; integer-mode data must match the oracle
exactly (R11), and the send lists bit-exactly.

Cases: flat P = 2 (both receive modes; single buffer; separate wait launch),
hierarchical P = 4 with groups of 2 (Algorithm 1's READY1 / READY2 /
CONSUMED protocol), an asymmetric P = 3 matrix where a rank
sends to a peer it receives nothing from (the step-end barrier), value refresh
and weighted plans across processes, a transposed plan, and a peer that never
signals (SHIRO_E_PEER after the timeout instead of a hang)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():   # pragma: no cover - CPU boxes
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(kind):
    import shiro_gen
    if kind == "c1":
        c = shiro_gen.CONFIGS["c1"]
        row_ptr, col, vi = shiro_gen.gen_matrix("c1", value_mode=1)
        return c.n, c.N, row_ptr, col, vi, c.seed
    # asymmetric P = 3 block pattern: A^(0,2) empty (rank 0 receives nothing
    # from rank 2) while A^(2,0) is not (rank 0 sends to rank 2)
    rng = np.random.default_rng(3)
    n, N = 900, 32
    m = rng.random((n, n)) < 0.01
    m[0:300, 600:900] = False
    rows, cols = np.nonzero(m)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return n, N, row_ptr, cols.astype(np.int32), rng.integers(1, 5, cols.size).astype(np.float32), 7


def _worker(rank, world, port, case, out_q):
    os.environ.update(case.get("env", {}))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("SHIRO_P2P_TIMEOUT_MS", "60000")
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2512_20178_b200 as sh
        import shiro_gen
        torch.cuda.set_device(0)
        n, N, row_ptr, col, vi, seed = _matrix(case.get("matrix", "c1"))
        flags, g = case.get("flags", 0), case.get("g", 1)
        part = oracle.uniform_partition(n, world)
        lo, hi = int(part[rank]), int(part[rank + 1])
        rp = row_ptr[lo:hi + 1] - row_ptr[lo]
        cl = col[row_ptr[lo]:row_ptr[hi]].copy()
        w = {}
        if case.get("weighted"):
            rng = np.random.default_rng(1)
            wr, wc = rng.integers(1, 6, n), rng.integers(1, 6, n)
            w = dict(w_row=wr[lo:hi], w_col=wc)
        pl = sh.Plan.distributed(rank, world, n, part, rp, cl, vi[row_ptr[lo]:row_ptr[hi]], N,
                                 group_size=g, flags=flags, host_xchg=sh.torch_dist_alltoallv(),
                                 **w)
        ok = True
        empty = np.empty(0, np.int64)
        if not flags & sh.F_TRANSPOSE:
            op = oracle.plan_flat(n, part, row_ptr, col,
                                  **({"w_row": wr, "w_col": wc} if w else {}))
            for p in range(world):
                if p != rank:
                    ok &= np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), empty))
                    ok &= np.array_equal(pl.list(p, sh.LIST_SEND_C), op.send_c.get((rank, p), empty))
        if case.get("silent_rank") == rank:
            dist.barrier()            # never calls shiro_spmm; waits for the peer's verdict
            out_q.put((rank, True, 0))
            return
        stream = torch.cuda.Stream()
        bad = 0
        vals = vi
        for step in range(case.get("steps", 5)):   # odd count: both receive buffers, twice each
            if case.get("refresh") and step == 2:
                vals = np.where(vi > 2, vi - 1, vi + 2).astype(np.float32)
                pl.update_values(vals[row_ptr[lo]:row_ptr[hi]], row_ptr=rp, col=cl, stream=stream)
            B = np.asarray(shiro_gen.gen_B(seed + 17 * step, 0, n, N, mode=1))
            if flags & sh.F_TRANSPOSE:
                rows = np.repeat(np.arange(n), np.diff(row_ptr))
                order = np.lexsort((rows, col))
                t_rp = np.zeros(n + 1, np.int64)
                np.cumsum(np.bincount(col, minlength=n), out=t_rp[1:])
                ref = oracle.spmm_ref(t_rp, rows[order], vals[order], B, rows=np.arange(lo, hi))
            else:
                ref = oracle.spmm_ref(row_ptr, col, vals, B, rows=np.arange(lo, hi))
            if case.get("silent_rank") is not None:
                Bh = torch.from_numpy(B[lo:hi].copy()).pin_memory()
                Ch = torch.empty((hi - lo, N)).pin_memory()
                try:
                    pl.spmm_host(Bh, Ch, stream)
                    out_q.put((rank, False, "no error from a silent peer"))
                except sh.ShiroError as e:
                    out_q.put((rank, e.code == 8, repr(e)))
                dist.barrier()
                return
            Bd = torch.from_numpy(B[lo:hi].copy()).cuda()
            Cd = torch.full((hi - lo, N), float("nan"), device="cuda")
            stream.wait_stream(torch.cuda.current_stream())   # B's copy and C's fill first
            with torch.cuda.stream(stream):
                pl.spmm(Bd, Cd, stream)
            stream.synchronize()
            bad += int((Cd.cpu().numpy().astype(np.float64) != ref).sum())
        out_q.put((rank, bool(ok), bad))
    except Exception as e:   # report instead of hanging the peer
        import traceback
        traceback.print_exc()
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, "worker hung or crashed"
    return sorted(q.get() for _ in range(world))


def _check(res):
    for rank, lists_ok, bad in res:
        assert lists_ok, (rank, bad)
        assert bad == 0, (rank, bad)


@pytest.mark.parametrize("env", [{}, {"SHIRO_DBUF": "0"}, {"SHIRO_INKERNEL_WAIT": "1"},
                                 {"SHIRO_INKERNEL_WAIT": "1", "SHIRO_DBUF": "0"},
                                 {"SHIRO_INKERNEL_WAIT": "1", "SHIRO_CX": "1"},
                                 {"SHIRO_INKERNEL_WAIT": "1", "SHIRO_CX": "1", "SHIRO_DBUF": "0"}],
                         ids=["default", "single-buffer", "per-unit-waits",
                              "per-unit-waits-single-buffer", "two-phase-consumer",
                              "two-phase-single-buffer"])
def test_two_process_fused_exchange_exact(env):
    import paper_2512_20178_b200 as sh
    for flags in (0, sh.F_SPLIT_RECV):
        _check(_run(2, {"flags": flags, "env": env}))


def test_four_process_hierarchical_exact():
    """Algorithm 1 across 4 processes (groups of 2): Stage I -> READY1 ->
    Stage II (pre-aggregation + forwarding from R1) -> READY2 -> final SpMM
    -> CONSUMED, 5 steps."""
    _check(_run(4, {"g": 2}))


def test_three_process_asymmetric_barrier():
    """Rank 0 sends to rank 2 but receives nothing from it: its consumer has
    no unit waiting on rank 2, so only the step-end barrier keeps it from
    overwriting rank 2's buffer of two steps ago too early."""
    _check(_run(3, {"matrix": "asym", "steps": 7}))


def test_two_process_refresh_weighted_transposed():
    import paper_2512_20178_b200 as sh
    _check(_run(2, {"refresh": True}))
    _check(_run(2, {"weighted": True, "refresh": True}))
    _check(_run(2, {"flags": sh.F_TRANSPOSE, "refresh": True}))


def test_silent_peer_reports_error_not_hang():
    """A peer that never runs its step: the waiting rank's kernels time out
    (shared error flag, one timeout however many waves) and shiro_spmm_host
    returns SHIRO_E_PEER."""
    res = _run(2, {"silent_rank": 1, "env": {"SHIRO_P2P_TIMEOUT_MS": "1500"}})
    for rank, ok, msg in res:
        assert ok, (rank, msg)
