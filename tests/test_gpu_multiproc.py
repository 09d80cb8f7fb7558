"""GPU: the multi-rank distributed path (shiro_plan / shiro_spmm with the fused
NVLink exchange) in two OS processes sharing cuda:0.

Each process is one rank: the plan-time exchange runs over gloo (caller
transport, no NCCL communicator), the per-step exchange is the fused one --
CUDA-IPC peer stores into the other process's receive buffer plus epoch
flags -- exactly the code the multi-GPU runs use, here on one device.
Several steps with different B exercise the double-buffered receive buffers
(the step parity alternates); integer-mode data must match the oracle
exactly (R11), and the send lists bit-exactly."""
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


def _worker(rank, world, port, flags, env, out_q):
    os.environ.update(env)
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
        c = shiro_gen.CONFIGS["c1"]
        row_ptr, col, vi = shiro_gen.gen_matrix("c1", value_mode=1)
        part = oracle.uniform_partition(c.n, world)
        lo, hi = int(part[rank]), int(part[rank + 1])
        rp = row_ptr[lo:hi + 1] - row_ptr[lo]
        pl = sh.Plan.distributed(rank, world, c.n, part, rp, col[row_ptr[lo]:row_ptr[hi]].copy(),
                                 vi[row_ptr[lo]:row_ptr[hi]], c.N, flags=flags,
                                 host_xchg=sh.torch_dist_alltoallv())
        op = oracle.plan_flat(c.n, part, row_ptr, col)
        ok = True
        empty = np.empty(0, np.int64)
        for p in range(world):
            if p != rank:
                ok &= np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), empty))
                ok &= np.array_equal(pl.list(p, sh.LIST_SEND_C), op.send_c.get((rank, p), empty))
        stream = torch.cuda.Stream()
        bad = 0
        for step in range(5):   # odd count: both receive buffers, twice each
            B = np.asarray(shiro_gen.gen_B(c.seed + 17 * step, 0, c.n, c.N, mode=1))
            ref = oracle.spmm_ref(row_ptr, col, vi, B, rows=np.arange(lo, hi))
            Bd = torch.from_numpy(B[lo:hi].copy()).cuda()
            Cd = torch.full((hi - lo, c.N), float("nan"), device="cuda")
            with torch.cuda.stream(stream):
                pl.spmm(Bd, Cd, stream)
            stream.synchronize()
            bad += int((Cd.cpu().numpy().astype(np.float64) != ref).sum())
        out_q.put((rank, bool(ok), bad))
    except Exception as e:   # report instead of hanging the peer
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, flags=0, env=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, flags, env or {}, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, "worker hung or crashed"
    return sorted(q.get() for _ in range(world))


@pytest.mark.parametrize("env", [{}, {"SHIRO_DBUF": "0"}, {"SHIRO_INKERNEL_WAIT": "0"}],
                         ids=["default", "single-buffer", "separate-wait-launch"])
def test_two_process_fused_exchange_exact(env):
    import paper_2512_20178_b200 as sh
    for flags in (0, sh.F_SPLIT_RECV):
        res = _run(2, flags, env)
        for rank, lists_ok, bad in res:
            assert lists_ok, (rank, bad)
            assert bad == 0, (rank, bad)
