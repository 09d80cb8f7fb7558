"""Multi-process planning over a real process group (gloo, CPU, world size 2
and 4): every rank calls shiro_plan with its own CSR rows and the plan-time
exchange runs through the caller's transport (torch.distributed over gloo).
Lists must equal the oracle's bit-exactly; a bad input on one rank must fail
every rank without a hang (status agreement before the payload exchange)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, bad_rank, out_q, weighted=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2512_20178_b200 as sh
    import shiro_gen
    try:
        c = shiro_gen.CONFIGS[cfg]
        row_ptr, col, val = shiro_gen.gen_matrix(cfg)
        part = oracle.uniform_partition(c.n, world)
        lo, hi = part[rank], part[rank + 1]
        rp = row_ptr[lo:hi + 1] - row_ptr[lo]
        cl = col[row_ptr[lo]:row_ptr[hi]].copy()
        vl = val[row_ptr[lo]:row_ptr[hi]]
        if rank == bad_rank and cl.size:
            cl[0] = c.n + 5                          # out of range column
        w = {}
        if weighted:      # N2: per-vertex costs (C rows of this rank, every B row)
            rng = np.random.default_rng(3)
            wr, wc = rng.integers(1, 9, c.n), rng.integers(1, 9, c.n)
            w = dict(w_row=wr[lo:hi], w_col=wc)
        try:
            pl = sh.Plan.distributed(rank, world, c.n, part, rp, cl, vl, c.N,
                                     flags=sh.F_HOST_ONLY, host_xchg=sh.torch_dist_alltoallv(),
                                     **w)
        except sh.ShiroError as e:
            out_q.put((rank, "error", e.code))
            return
        op = oracle.plan_flat(c.n, part, row_ptr, col,
                              **({"w_row": wr, "w_col": wc} if weighted else {}))
        ok = True
        empty = np.empty(0, np.int64)
        for p in range(world):
            if p == rank:
                continue
            ok &= np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), empty))
            ok &= np.array_equal(pl.list(p, sh.LIST_SEND_C), op.send_c.get((rank, p), empty))
            ok &= np.array_equal(pl.list(p, sh.LIST_RECV_B), op.send_b.get((p, rank), empty))
            ok &= np.array_equal(pl.list(p, sh.LIST_RECV_C), op.send_c.get((p, rank), empty))
        info = pl.info()
        vol = oracle.volumes(op, c.N)
        ok &= info["g_joint_rows"] == vol["joint_rows"] and info["g_col_rows"] == vol["col_rows"]
        out_q.put((rank, "ok" if ok else "mismatch", 0))
    finally:
        dist.destroy_process_group()


def _run(world, cfg, bad_rank=-1, weighted=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, bad_rank, q, weighted))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, "worker hung or crashed"
    return sorted(q.get() for _ in range(world))


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_distributed_plan_matches_oracle(world):
    res = _run(world, "c1")
    assert all(r[1] == "ok" for r in res), res


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_weighted_plan_matches_oracle(world):
    """Weighted covers (N2) planned by separate processes over gloo."""
    res = _run(world, "c1", weighted=True)
    assert all(r[1] == "ok" for r in res), res


def test_gloo_bad_input_fails_every_rank():
    res = _run(2, "c1", bad_rank=1)
    assert res[0][1] == "error" and res[0][2] == 8        # SHIRO_E_PEER on the good rank
    assert res[1][1] == "error" and res[1][2] == 2        # SHIRO_E_CSR on the bad rank
