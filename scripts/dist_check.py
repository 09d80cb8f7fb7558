"""Multi-GPU correctness of the distributed path (one process per GPU, NCCL).

    torchrun --nproc-per-node P --master-addr 127.0.0.1 --master-port 29511 \
        scripts/dist_check.py --config c2 [--flags split,colmax] [--int]

Every rank plans with shiro_plan (NCCL plan-time exchange), runs shiro_spmm
(NCCL all-to-allv), and rank 0 checks the gathered C against the CPU oracle
(tolerance of DESIGN.md R11, exact in integer mode) and every rank's lists
against the oracle plan bit-exactly.  Prints one JSON line on rank 0.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2512_20178_b200 as sh  # noqa: E402
import shiro_gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--flags", default="")
    ap.add_argument("--int", action="store_true")
    ap.add_argument("--group-size", type=int, default=1)
    ap.add_argument("--sample", type=int, default=0, help="check only this many C rows")
    ap.add_argument("--no-lists", action="store_true",
                    help="skip the oracle plan (its Dinic over every block is slow at c5 size)")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = shiro_gen.CONFIGS[args.config]
    vm = 1 if args.int else 0
    row_ptr, col, val = shiro_gen.gen_matrix_shared(cfg, rank, dist.barrier, value_mode=vm)
    part = sh.uniform_partition(cfg.n, world)
    lo, hi = int(part[rank]), int(part[rank + 1])
    rp_l, col_l, val_l = sh.local_rows(row_ptr, col, val, part, rank)
    flags = 0
    for f in filter(None, args.flags.split(",")):
        flags |= {"split": sh.F_SPLIT_RECV, "colmax": sh.F_COVER_COLMAX, "col": sh.F_MODE_COL,
                  "row": sh.F_MODE_ROW, "nooverlap": sh.F_NO_OVERLAP, "nccl": sh.F_XCHG_NCCL,
                  "balance": sh.F_COVER_BALANCE}[f]
    obj = [sh.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    pl = sh.Plan.distributed(rank, world, cfg.n, part, rp_l, col_l, val_l, cfg.N,
                             group_size=args.group_size, flags=flags, nccl_id=obj[0])
    B_p = shiro_gen.gen_B(cfg.seed, lo, hi - lo, cfg.N, mode=vm)
    Bd = torch.from_numpy(B_p).to(dev)
    Cd = torch.full((hi - lo, cfg.N), float("nan"), device=dev)
    for _ in range(2):                     # twice: buffers are reused across calls
        pl.spmm(Bd, Cd)
    torch.cuda.synchronize()
    # lists vs oracle (every rank checks its own)
    op = None if args.no_lists else oracle.plan_flat(cfg.n, part, row_ptr, col,
                          mode="col" if flags & sh.F_MODE_COL else "row" if flags & sh.F_MODE_ROW else "joint",
                          rule="colmax" if flags & sh.F_COVER_COLMAX else "rowmax",
                          balance=bool(flags & sh.F_COVER_BALANCE))
    empty = np.empty(0, np.int64)
    lists_ok = True
    for p in range(world if op is not None else 0):
        if p == rank:
            continue
        lists_ok &= np.array_equal(pl.list(p, sh.LIST_SEND_B), op.send_b.get((rank, p), empty))
        lists_ok &= np.array_equal(pl.list(p, sh.LIST_SEND_C), op.send_c.get((rank, p), empty))
        lists_ok &= np.array_equal(pl.list(p, sh.LIST_RECV_B), op.send_b.get((p, rank), empty))
        lists_ok &= np.array_equal(pl.list(p, sh.LIST_RECV_C), op.send_c.get((p, rank), empty))
    # gather C on rank 0
    sizes = [int(part[r + 1] - part[r]) for r in range(world)]
    mx = max(sizes)
    Cpad = torch.zeros((mx, cfg.N), device=dev)      # NCCL gather needs equal sizes
    Cpad[:hi - lo] = Cd
    if rank == 0:
        parts = [torch.empty((mx, cfg.N), device=dev) for _ in sizes]
        dist.gather(Cpad, parts, dst=0)
        parts = [t[:s] for t, s in zip(parts, sizes)]
    else:
        dist.gather(Cpad, None, dst=0)
    ok_t = torch.tensor([1 if lists_ok else 0], device=dev)
    dist.all_reduce(ok_t, op=dist.ReduceOp.MIN)
    if rank == 0:
        C = torch.cat(parts).cpu().numpy()
        rows = None
        if args.sample:
            rows = np.unique(np.random.default_rng(0).integers(0, cfg.n, args.sample)).astype(np.int64)
            # only the B rows the sampled rows reference (c5: B is 17 GB)
            starts, ends = row_ptr[rows], row_ptr[rows + 1]
            idx = np.concatenate([np.arange(a, b) for a, b in zip(starts, ends)]).astype(np.int64)
            ucols = np.unique(col[idx])
            Bs = np.concatenate([shiro_gen.gen_B(cfg.seed, int(c), 1, cfg.N, mode=vm) for c in ucols]) \
                if ucols.size else np.zeros((0, cfg.N), np.float32)
            srp = np.concatenate([[0], np.cumsum(ends - starts)]).astype(np.int64)
            ref = oracle.spmm_ref(srp, np.searchsorted(ucols, col[idx]).astype(np.int32), val[idx], Bs)
        else:
            B = shiro_gen.gen_B(cfg.seed, 0, cfg.n, cfg.N, mode=vm)
            ref = oracle.spmm_ref(row_ptr, col, val, B)
        got = C if rows is None else C[rows]
        d = np.abs(got.astype(np.float64) - ref)
        bad = int((d > np.maximum(1e-4 * np.abs(ref), 1e-6)).sum()) if not args.int else \
            int((d != 0).sum())
        info = pl.info()
        print(json.dumps({"config": args.config, "P": world, "flags": args.flags, "int": args.int,
                          "lists_bit_exact": bool(ok_t.item()), "bad_elements": bad,
                          "checked_rows": int(got.shape[0]), "max_abs_err": float(d.max()),
                          "joint_rows": info["g_joint_rows"], "oblivious_rows": info["g_oblivious_rows"],
                          "plan_seconds": round(info["plan_seconds"], 3)}), flush=True)
    pl.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
