"""Step-wise ablation and communication-pattern heatmaps:
the shape of the paper's volume, heatmap and
step-wise runtime figures on the synthetic configs.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 --master-port 29511 \
        scripts/ablation.py --config c4 [--group-size 2] [--out gpurun_out/ablation_c4]

For each strategy -- block (sparsity-oblivious, Eq. 1), col (Eq. 2), row
(Eq. 3), joint (SHIRO), joint + hierarchy -- plans with shiro_plan, times K
steps of shiro_spmm (graph replays, L2 flushed, max over ranks) and records
the rows each rank sends to each peer.  Rank 0 writes <out>.json (one record
per strategy) and <out>_<strategy>_pairs.csv (P x P bytes, row = source,
normalised by the maximum as in the paper's heatmaps, plus raw bytes).
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
import paper_2512_20178_b200 as sh  # noqa: E402
import shiro_gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--group-size", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/ablation")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = shiro_gen.CONFIGS[args.config]
    row_ptr, col, val = shiro_gen.gen_matrix_shared(cfg, rank, dist.barrier)
    part = sh.uniform_partition(cfg.n, world)
    lo, hi = int(part[rank]), int(part[rank + 1])
    rp_l, col_l, val_l = sh.local_rows(row_ptr, col, val, part, rank)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    Bd = torch.from_numpy(shiro_gen.gen_B(cfg.seed, lo, hi - lo, cfg.N)).to(dev)
    Cd = torch.empty_like(Bd)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    only = set(filter(None, os.environ.get("ABLATION_ONLY", "").split(",")))
    strategies = [("block", sh.F_MODE_BLOCK, 1), ("col", sh.F_MODE_COL, 1),
                  ("row", sh.F_MODE_ROW, 1), ("joint", 0, 1),
                  ("joint-colmax", sh.F_COVER_COLMAX, 1),
                  ("joint-balanced", sh.F_COVER_BALANCE, 1)]
    if args.group_size > 1 and world % args.group_size == 0 and world > args.group_size:
        strategies.append((f"joint+hier(g={args.group_size})", 0, args.group_size))
    records = []
    for name, flags, g in strategies:
        if only and name.split("(")[0] not in only:
            continue
        obj = [sh.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        pl = sh.Plan.distributed(rank, world, cfg.n, part, rp_l, col_l, val_l, cfg.N,
                                 group_size=g, flags=flags, nccl_id=obj[0], stream=stream)
        for _ in range(3):
            pl.spmm(Bd, Cd, stream)
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pl.spmm(Bd, Cd, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = torch.tensor(ts, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # rows this rank sends to every peer (flat lists; for the hierarchical
        # schedule the stage-I + stage-II lists)
        sent = np.zeros(world, np.int64)
        for p in range(world):
            if p == rank:
                continue
            if g > 1:
                sent[p] = pl.list(p, sh.LIST_H1_SEND).size + pl.list(p, sh.LIST_H2_SEND).size
            else:
                sent[p] = pl.list(p, sh.LIST_SEND_B).size + pl.list(p, sh.LIST_SEND_C).size
        mat = torch.from_numpy(sent).to(dev)
        allm = [torch.zeros_like(mat) for _ in range(world)]
        dist.all_gather(allm, mat)
        info = pl.info()
        if rank == 0:
            pairs = np.stack([m.cpu().numpy() for m in allm]) * 4 * cfg.N     # bytes, row = source
            tag = name.split("(")[0].replace("+", "_")
            mx = pairs.max() if pairs.max() > 0 else 1
            with open(f"{args.out}_{tag}_pairs.csv", "w") as f:
                f.write("# bytes sent per (source row, destination column); normalised, then raw\n")
                for r in range(world):
                    f.write(",".join(f"{x / mx:.4f}" for x in pairs[r]) + "\n")
                for r in range(world):
                    f.write(",".join(str(int(x)) for x in pairs[r]) + "\n")
            grp = np.arange(world) // max(g, 1) if g > 1 else np.arange(world) // args.group_size
            inter = int(sum(pairs[s, d] for s in range(world) for d in range(world)
                            if grp[s] != grp[d]))
            rec = {"strategy": name, "config": cfg.name, "P": world, "N": cfg.N,
                   "ms_per_step": round(float(t.mean().item()), 5),
                   "gflops": round(2 * int(row_ptr[-1]) * cfg.N / (float(t.mean().item()) * 1e-3) / 1e9, 1),
                   "bytes_total": int(pairs.sum()),
                   "bytes_inter_group": inter,
                   "oblivious_allgather_bytes": info["g_oblivious_rows"] * 4 * cfg.N,
                   "max_pair_over_mean": round(float(pairs.max() / max(pairs[pairs > 0].mean(), 1)), 3),
                   "plan_seconds": round(info["plan_seconds"], 3)}
            records.append(rec)
            print(json.dumps(rec), flush=True)
        pl.free()
    if rank == 0:
        json.dump(records, open(f"{args.out}.json", "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
