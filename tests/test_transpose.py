"""Transposed SpMM: SHIRO_F_TRANSPOSE plans A^T from the
ranks' rows of A (one distributed transpose at plan time).  The oracle side
transposes with numpy and runs its own plan on A^T; lists must match
bit-exactly and the product must be A^T B."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_2512_20178_b200 as sh
from conftest import random_csr
from test_planner_parity import assert_lists_equal


def csr_transpose(n, row_ptr, col, val):
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    order = np.lexsort((rows, col))
    t_rows, t_cols, t_val = col[order].astype(np.int64), rows[order], val[order]
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(t_rows, minlength=n), out=rp[1:])
    return rp, t_cols.astype(np.int32), t_val


@pytest.mark.parametrize("P,seed", [(1, 0), (2, 1), (4, 2), (8, 3)])
def test_loopback_transpose_lists(P, seed):
    rng = np.random.default_rng(900 + seed)
    n = 250
    row_ptr, col, val = random_csr(rng, n, 0.03)
    part = oracle.uniform_partition(n, P)
    pl = sh.Plan.loopback(P, n, part, row_ptr, col, val, 8, flags=sh.F_TRANSPOSE | sh.F_HOST_ONLY)
    trp, tcol, tval = csr_transpose(n, row_ptr, col, val)
    op = oracle.plan_flat(n, part, trp, tcol)
    assert_lists_equal(pl, op, P)
    assert pl.info()["nnz_local"] == int(trp[part[1]] - trp[0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        n = 300
        row_ptr, col, val = random_csr(rng, n, 0.03)
        part = oracle.uniform_partition(n, world)
        rp, cl, vl = sh.local_rows(row_ptr, col, val, part, rank)
        pl = sh.Plan.distributed(rank, world, n, part, rp, cl, vl, 8,
                                 flags=sh.F_TRANSPOSE | sh.F_HOST_ONLY,
                                 host_xchg=sh.torch_dist_alltoallv())
        trp, tcol, _ = csr_transpose(n, row_ptr, col, val)
        op = oracle.plan_flat(n, part, trp, tcol)
        e = np.empty(0, np.int64)
        ok = all(np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), e)) and
                 np.array_equal(pl.list(p, sh.LIST_RECV_C), op.send_c.get((p, rank), e))
                 for p in range(world) if p != rank)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_distributed_transpose():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(3))
    assert all(ok for _, ok in res), res
