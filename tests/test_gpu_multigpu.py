"""GPU, two or more devices: the distributed path with one process per GPU,
NCCL communicators and NVLink -- the NCCL grouped send/recv exchange
(SHIRO_F_XCHG_NCCL) next to the default fused exchange, and
the hierarchical schedule across physical GPUs.  Skipped on single-GPU boxes
(the single-GPU multi-process suite in test_gpu_multiproc.py covers the fused
protocol there); run with `gpurun --gpus 2` / `--gpus 4`.

Integer-mode data, 5 steps, exact against the oracle (R11); send
lists bit-exact."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:   # pragma: no cover
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, flags, g, cfg_name, env, out_q):
    os.environ.update(env)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("SHIRO_P2P_TIMEOUT_MS", "60000")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import oracle
        import paper_2512_20178_b200 as sh
        import shiro_gen
        c = shiro_gen.CONFIGS[cfg_name]
        row_ptr, col, _ = shiro_gen.gen_matrix(cfg_name)
        vi = shiro_gen.gen_values(cfg_name, row_ptr, col, 1)
        part = oracle.uniform_partition(c.n, world)
        lo, hi = int(part[rank]), int(part[rank + 1])
        obj = [sh.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rp = row_ptr[lo:hi + 1] - row_ptr[lo]
        pl = sh.Plan.distributed(rank, world, c.n, part, rp, col[row_ptr[lo]:row_ptr[hi]].copy(),
                                 vi[row_ptr[lo]:row_ptr[hi]], c.N, group_size=g, flags=flags,
                                 nccl_id=obj[0])
        op = oracle.plan_flat(c.n, part, row_ptr, col)
        ok = True
        empty = np.empty(0, np.int64)
        for p in range(world):
            if p != rank:
                ok &= np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), empty))
                ok &= np.array_equal(pl.list(p, sh.LIST_SEND_C), op.send_c.get((rank, p), empty))
        stream = torch.cuda.Stream()
        bad = 0
        for step in range(5):
            B = np.asarray(shiro_gen.gen_B(c.seed + 31 * step, lo, hi - lo, c.N, mode=1))
            Bfull = np.asarray(shiro_gen.gen_B(c.seed + 31 * step, 0, c.n, c.N, mode=1))
            ref = oracle.spmm_ref(row_ptr, col, vi, Bfull, rows=np.arange(lo, hi))
            Bd = torch.from_numpy(B).cuda()
            Cd = torch.full((hi - lo, c.N), float("nan"), device="cuda")
            stream.wait_stream(torch.cuda.current_stream())   # B's copy and C's fill first
            pl.spmm(Bd, Cd, stream)
            stream.synchronize()
            bad += int((Cd.cpu().numpy().astype(np.float64) != ref).sum())
        out_q.put((rank, bool(ok), bad))
    except Exception as e:
        import traceback
        traceback.print_exc()
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, flags, g=1, cfg="c2", env=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, flags, g, cfg, env or {}, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
        assert p.exitcode == 0, "worker hung or crashed"
    res = sorted(q.get() for _ in range(world))
    for rank, lists_ok, bad in res:
        assert lists_ok, (rank, bad)
        assert bad == 0, (rank, bad)


@pytest.mark.parametrize("flags", ["fused", "fused-two-phase", "fused-per-unit-waits", "nccl",
                                   "nccl-split"])
def test_two_gpus_exchanges_exact(flags):
    import paper_2512_20178_b200 as sh
    f = {"nccl": sh.F_XCHG_NCCL, "nccl-split": sh.F_XCHG_NCCL | sh.F_SPLIT_RECV}.get(flags, 0)
    env = {"fused-two-phase": {"SHIRO_INKERNEL_WAIT": "1", "SHIRO_CX": "1",
                               "SHIRO_P2P_TIMEOUT_MS": "20000"},
           "fused-per-unit-waits": {"SHIRO_INKERNEL_WAIT": "1"}}.get(flags, {})
    _run(2, f, env=env)


def test_four_gpus_flat_and_hierarchical_exact():
    if torch.cuda.device_count() < 4:
        pytest.skip("needs 4 GPUs")
    _run(4, 0)
    _run(4, 0, env={"SHIRO_INKERNEL_WAIT": "1"})
    _run(4, 0, env={"SHIRO_INKERNEL_WAIT": "1", "SHIRO_CX": "1", "SHIRO_P2P_TIMEOUT_MS": "20000"})
    _run(4, 0, g=2)
