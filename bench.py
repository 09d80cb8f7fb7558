#!/usr/bin/env python
"""Benchmark of the SHIRO distributed SpMM hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--also c4]
                    [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

A step = one shiro_spmm (all of DESIGN.md rows E1-E6) over the config's
synthetic matrix, 1D row-partitioned over the N ranks (P = N), with B and C
resident in HBM.  The plan (rows P1-P4) is built once before timing (PAPER.md
L300: "performed offline ... reused across multiple SpMM operations").
L2 is flushed (a 256 MiB device memset) before every timed step; each step is
bracketed by synchronize + barrier and timed with CUDA events on the
launching stream; the per-step time is the max over ranks.

The headline workload is c3 (the largest configuration that fits one GPU with
the most FLOPs); c4 is measured in the same run and reported
under "also".  Prints ONE JSON line on rank 0 (DESIGN.md section 6 lists every
field).  Roofline denominators are measured in the same run (FP32 FMA probe,
float4 HBM copy probe, NVLink peer-store probe at N > 1) next to the
driver-written MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "SpMM GFLOP/s (2·nnz·N) at 1/2/4/8 B200 + bytes communicated vs oblivious"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return dict(PEAKS_FALLBACK)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms (from the
    warm-up through the timed region, the attribution pass and the e2e pass)."""
    Q = ("index,clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = str(gpu_index)
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "50", "-i", self.gpu], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        busy = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit() and
                r[3].isdigit() and int(r[3]) > 0]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(busy or sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "samples_busy": len(busy)}


# ----------------------------------------------------------------- roofline
def op_bytes(info, N, op):
    """Algorithmic (compulsory) HBM bytes of one launch of device op `op`
    (DESIGN.md section 5): CSR index+value 8 B per nonzero, row_ptr 8 B per
    row, out_row 4 B per row, every distinct source row read once (4N B),
    every output row written once (4N B), accumulating ops also read it."""
    z, r, s = info["op_nnz"][op], info["op_rows"][op], info["op_src_rows"][op]
    row = 4 * N
    if op == "pack":
        return 8 * r + row * s + row * r
    if op == "scatter":
        return 12 * r + 4 * z + row * s + 2 * row * r
    b = 8 * z + 8 * (r + 1) + row * s + row * r
    if op != "local":
        b += 4 * r                       # out_row map / per-row output pointer
    if op == "remote":
        b += row * r                     # C read-modify-write
    return b


STAGE_OF_OP = {"local": "local", "partial": "partial", "remote": "remote",
               "scatter": "scatter", "pack": "pack"}


def step_terms(info, N):
    """SURVEY 8(d) per-rank terms of one step: algorithmic HBM bytes, FP32
    flops and NVLink bytes (max of sent and received rows)."""
    M = info["m_local"]
    nnz_g = info["nnz_diag"] + info["nnz_colbased"] + info["nnz_rowbased_computed"]
    send = info["send_b_rows"] + info["send_c_rows"]
    recv = info["recv_b_rows"] + info["recv_c_rows"]
    hbm = 8 * nnz_g + 4 * (M + 1) + 4 * N * M + 4 * N * M + 4 * N * send + 2 * 4 * N * recv
    flop = 2 * N * nnz_g + N * info["recv_c_rows"]
    nvl = 4 * N * max(send, recv)
    return [float(hbm), float(flop), float(nvl), float(nnz_g), float(send), float(recv)]


def traffic_from_profiles(config, world, op):
    """dram bytes per launch from a committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{config}/P{world}/{op}")


def bytes_table():
    p = os.path.join(ROOT, "profiles", "bytes_table.json")
    if not os.path.exists(p):
        return None
    return {"source": "host-only plans, scripts/bytes_table.py (profiles/bytes_table.json)",
            "rows": json.load(open(p))}


# ----------------------------------------------------------------- NVLink counters
def nvlink_bytes(gpu_index):
    """(tx, rx) NVLink data bytes of this GPU since boot, summed over links,
    from NVML's throughput counters (KiB); None where unsupported."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        tx = rx = 0
        got = False
        for link in range(18):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(
                    h, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                        (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
            except Exception:
                break
            if v[0].nvmlReturn == 0 and v[1].nvmlReturn == 0:
                tx += v[0].value.ullVal
                rx += v[1].value.ullVal
                got = True
        if got:
            return (tx * 1024, rx * 1024)
    except Exception:
        pass
    # fallback: `nvidia-smi nvlink -gt d` (per-link "Tx"/"Rx" data counters, KiB)
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(gpu_index)],
                             capture_output=True, text=True, timeout=20).stdout
        import re
        tx = rx = 0
        got = False
        for line in out.splitlines():
            m = re.search(r"(Tx|Rx)[^0-9]*([0-9]+)", line)
            if m:
                got = True
                if m.group(1) == "Tx":
                    tx += int(m.group(2))
                else:
                    rx += int(m.group(2))
        return (tx * 1024, rx * 1024) if got else None
    except Exception:
        return None


# ----------------------------------------------------------------- probes
def timed(fn, stream, torch, reps=5, flush=None):
    ts = []
    fn()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def probe_peaks(sh, torch, dev, stream):
    """FP32 FMA and HBM copy rates of this GPU, measured live."""
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 4096
    out = torch.empty(blocks * 256, device=dev)
    ms = timed(lambda: sh.probe_fma(out, blocks, iters, stream), stream, torch)
    fp32 = blocks * 256 * iters * 64 / (ms * 1e-3) / 1e12
    n = 1 << 28                                   # 1 GiB per buffer
    x = torch.ones(n, device=dev)
    y = torch.empty_like(x)
    ms_c = timed(lambda: sh.probe_copy(x, y, stream), stream, torch)
    copy = 8 * n / (ms_c * 1e-3) / 1e9
    del x, y
    return {"fp32_tflops": round(fp32, 2), "copy_gbs": round(copy, 1), "sms": sms}


def gather_probes(sh, torch, dev, stream, Bd, col_l, lo, hi, N, flush, reps=5):
    if N not in (32, 64, 128):
        return None
    res = {}

    def timeit(X, idx):
        out = torch.empty(((idx.numel() + 255) // 256, N), device=dev)
        ms = timed(lambda: sh.probe_gather(X, idx, out, 256, stream), stream, torch, reps, flush)
        return ms, idx.numel() * N * 4 / (ms * 1e-3) / 1e9

    # the local SpMM's own diagonal-block column stream (CSR order)
    c = np.asarray(col_l, np.int64)
    keep = (c >= lo) & (c < hi)
    idx = torch.from_numpy((c[keep] - lo).astype(np.int32)).to(dev)
    if idx.numel():
        ms, gbs = timeit(Bd, idx)
        res["csr_stream_ms"] = round(ms, 5)
        res["csr_stream_gbs"] = round(gbs, 1)
    g = torch.Generator(device="cpu").manual_seed(0)
    n_idx = 1 << 22
    for name, rows in (("l2_random_gbs", (32 << 20) // (4 * N)), ("hbm_random_gbs", (4 << 30) // (4 * N))):
        X = torch.ones((rows, N), device=dev)
        ridx = torch.randint(0, rows, (n_idx,), generator=g, dtype=torch.int32).to(dev)
        res[name] = round(timeit(X, ridx)[1], 1)
        del X
    return res


def perm_matrix(n, part, rank, k):
    """This rank's rows of the NVLink probe matrix: row part[p]+i (i < k) has
    one nonzero in every other block, column part[q]+i (a perfect matching per
    block, so every block's canonical cover is its k rows and q ships k rows
    of N floats to p)."""
    P = part.size - 1
    lo, hi = int(part[rank]), int(part[rank + 1])
    rows = []
    for t in range(lo, hi):
        i = t - lo
        rows.append([int(part[q]) + i for q in range(P) if q != rank and i < k])
    rp = np.zeros(hi - lo + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.array([c for r in rows for c in r], np.int32)
    return rp, col, np.ones(col.size, np.float32)


def nvlink_probe(sh, torch, dist, dev, stream, world, rank, nccl_id, N=128, k=1 << 17):
    """Per-direction NVLink bandwidth of (a) the fused exchange's own peer
    stores (producer launch of a plan whose every block is a k-row perfect
    matching: k(P-1) rows of 4N B stored into peers, timed with the plan's
    stage events) and (b) NCCL all_to_all_single of the same bytes."""
    n = world * k
    part = sh.uniform_partition(n, world)
    rp, col, val = perm_matrix(n, part, rank, k)
    pl = sh.Plan.distributed(rank, world, n, part, rp, col, val, N, nccl_id=nccl_id,
                             flags=sh.F_MODE_COL)
    Bd = torch.ones((k, N), device=dev)
    Cd = torch.empty((k, N), device=dev)
    for _ in range(3):
        pl.spmm(Bd, Cd, stream)
    torch.cuda.synchronize()
    pl.profile(True)
    prod = []
    for _ in range(10):
        dist.barrier()
        pl.spmm(Bd, Cd, stream)
        torch.cuda.synchronize()
        prod.append(pl.stage_times()["partial"])
    pl.profile(False)
    pl.free()
    nbytes = (world - 1) * k * N * 4
    ms = float(np.median(prod))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ipc = nbytes / (t.item() * 1e-3) / 1e9
    # NCCL all-to-all of the same per-rank bytes
    send = torch.ones(world * k * N, device=dev)
    recv = torch.empty_like(send)
    for _ in range(3):
        dist.all_to_all_single(recv, send)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.all_to_all_single(recv, send)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t2 = torch.tensor([float(np.median(ts))], dtype=torch.float64, device=dev)
    dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    nccl = nbytes / (t2.item() * 1e-3) / 1e9
    del send, recv
    return {"ipc_store_gbs": round(ipc, 1), "nccl_alltoall_gbs": round(nccl, 1),
            "bytes_per_rank": nbytes, "producer_ms": round(t.item(), 5),
            "how": f"k={k} rows x N={N} fp32 to each of {world - 1} peers per rank; "
                   "per-direction bytes / max-over-ranks time"}


def t_floor(sh, torch, dist, dev, stream, world, rank, nccl_id, N, barrier):
    """Latency floor of one step: 1 row per non-empty pair and
    1 nonzero per row at the same P and N."""
    k = 1
    n = world * 64
    part = sh.uniform_partition(n, world)
    rp, col, val = perm_matrix(n, part, rank, k)
    pl = sh.Plan.distributed(rank, world, n, part, rp, col, val, N, nccl_id=nccl_id)
    Bd = torch.ones((64, N), device=dev)
    Cd = torch.empty((64, N), device=dev)
    for _ in range(5):
        pl.spmm(Bd, Cd, stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pl.spmm(Bd, Cd, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    pl.free()
    t = torch.tensor(ts, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(float(t.median().item()), 5)


# ----------------------------------------------------------------- reference arm
def run_reference(args, cfg, world, rank):
    """The oracle (as it stands) on the host cores: each step computes the
    fp64 product of a bounded row sample of the same matrix."""
    if rank != 0:
        return
    import oracle
    import shiro_gen
    row_ptr, col, val = shiro_gen.gen_matrix(cfg, cache_dir=_cache_dir())
    B = shiro_gen.gen_B(cfg.seed, 0, cfg.n, cfg.N)
    rows, nnz_s = _sample_rows(row_ptr, budget_nnz=1_500_000)
    cores = os.cpu_count()
    for _ in range(args.warmup):
        oracle.spmm_ref(row_ptr, col, val, B, rows=rows)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.spmm_ref(row_ptr, col, val, B, rows=rows)
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    v = 2 * nnz_s * cfg.N / t / 1e9
    sample = f"{rows.size} of {cfg.n} rows ({nnz_s} of {int(row_ptr[-1])} nnz), fp64 oracle"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "n": cfg.n, "nnz": cfg.nnz,
                   "N": cfg.N, "P": world},
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def _sample_rows(row_ptr, budget_nnz):
    """Evenly strided rows whose nonzeros total about budget_nnz (all rows if
    the matrix is smaller)."""
    n = row_ptr.size - 1
    nnz = int(row_ptr[-1])
    if nnz <= budget_nnz:
        rows = np.arange(n, dtype=np.int64)
    else:
        stride = max(1, int(np.ceil(nnz / budget_nnz)))
        rows = np.arange(0, n, stride, dtype=np.int64)
    deg = row_ptr[rows + 1] - row_ptr[rows]
    return rows, int(deg.sum())


def _cache_dir():
    return os.environ.get("SHIRO_GEN_CACHE", "/tmp/shiro_gen_cache")


def cpu_baseline(cfg, row_ptr, col, val, B_full, target_s=10.0):
    """The oracle's fp64 product on the host cores (rank 0, N=1 only): a row
    sample of the matrix repeated for about target_s seconds."""
    import oracle
    rows, nnz_s = _sample_rows(row_ptr, budget_nnz=20_000_000)
    t0 = time.perf_counter()
    oracle.spmm_ref(row_ptr, col, val, B_full, rows=rows)
    t1 = time.perf_counter() - t0
    reps = max(1, int(target_s / max(t1, 1e-3)))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.spmm_ref(row_ptr, col, val, B_full, rows=rows)
    t = (time.perf_counter() - t0) / reps
    return {"value": round(2 * nnz_s * cfg.N / t / 1e9, 3), "unit": "GFLOP/s",
            "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{rows.size} of {cfg.n} rows ({nnz_s} nnz) x {reps} repetitions, "
                      f"fp64 accumulation, OpenMP over rows, {t * reps:.1f} s total"}


# ----------------------------------------------------------------- one config
def measure(cfg_name, args, ctx, primary):
    """Plan + timed steps + attribution pass + rooflines of one config."""
    import shiro_gen
    sh, torch, dist = ctx["sh"], ctx["torch"], ctx["dist"]
    world, rank, dev, stream = ctx["world"], ctx["rank"], ctx["dev"], ctx["stream"]
    barrier = ctx["barrier"]
    cfg = shiro_gen.CONFIGS[cfg_name]
    row_ptr, col, val = shiro_gen.gen_matrix_shared(cfg, rank, barrier, cache_dir=_cache_dir())
    nnz = int(row_ptr[-1])
    part = sh.uniform_partition(cfg.n, world)
    lo, hi = int(part[rank]), int(part[rank + 1])
    M = hi - lo
    rp_l, col_l, val_l = sh.local_rows(row_ptr, col, val, part, rank)
    B_p = shiro_gen.gen_B(cfg.seed, lo, M, cfg.N)

    flags = 0
    if args.split_recv:
        flags |= sh.F_SPLIT_RECV
    if args.colmax:
        flags |= sh.F_COVER_COLMAX
    if args.balance:
        flags |= sh.F_COVER_BALANCE
    flags |= {"joint": 0, "col": sh.F_MODE_COL, "row": sh.F_MODE_ROW}[args.mode]
    if args.xchg == "nccl":
        flags |= sh.F_XCHG_NCCL
    plan = sh.Plan.distributed(rank, world, cfg.n, part, rp_l, col_l, val_l, cfg.N,
                               group_size=args.group_size, flags=flags, nccl_id=ctx["fresh_id"]())
    info = plan.info()

    Bd = torch.from_numpy(B_p).to(dev)
    Cd = torch.empty((M, cfg.N), device=dev)
    flush = ctx["flush"]
    for _ in range(args.warmup):
        plan.spmm(Bd, Cd, stream)
    torch.cuda.synchronize()
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    step_ms, stages = [], []
    launches = 0
    nvl0 = nvlink_bytes(ctx["local"]) if world > 1 else None
    # timed region: K steps (each a CUDA-graph replay of shiro_spmm)
    for k in range(args.steps):
        flush.zero_()                                   # L2 flush, outside the timed window
        torch.cuda.synchronize()
        barrier()
        ev[k][0].record(stream)
        plan.spmm(Bd, Cd, stream)
        ev[k][1].record(stream)
        torch.cuda.synchronize()
        step_ms.append(ev[k][0].elapsed_time(ev[k][1]))
        launches += plan.last_launches()
    nvl1 = nvlink_bytes(ctx["local"]) if world > 1 else None
    barrier()
    # attribution pass: the same schedule with per-stage CUDA events (direct
    # launches on the same streams) -> which kernel dominates and its duration
    plan.profile(True)
    for k in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        plan.spmm(Bd, Cd, stream)
        torch.cuda.synchronize()
        stages.append(plan.stage_times())
    plan.profile(False)

    # max over ranks, per step and per stage
    t = torch.tensor(step_ms, dtype=torch.float64, device=dev)
    st = torch.tensor([[s[x] for x in sh.STAGES] for s in stages], dtype=torch.float64, device=dev)
    terms = torch.tensor(step_terms(info, cfg.N), dtype=torch.float64, device=dev)
    per_rank, all_terms = None, [terms]
    if world > 1:
        mine = st.mean(0)
        allr = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = [{k: round(v, 4) for k, v in zip(sh.STAGES, r.cpu().numpy().tolist()) if v}
                    for r in allr]
        wk = torch.tensor([float(info["op_nnz"][op]) for op in sh.OPS], dtype=torch.float64,
                          device=dev)
        allw = [torch.empty_like(wk) for _ in range(world)]
        dist.all_gather(allw, wk)
        for d_, w_ in zip(per_rank, allw):
            d_["op_nnz"] = {op: int(x) for op, x in zip(sh.OPS, w_.cpu().numpy().tolist()) if x}
        all_terms = [torch.empty_like(terms) for _ in range(world)]
        dist.all_gather(all_terms, terms)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(st, op=dist.ReduceOp.MAX)
    step_ms = t.cpu().numpy()
    stage_ms = dict(zip(sh.STAGES, st.mean(0).cpu().numpy().tolist()))
    ms = float(step_ms.mean())
    value = 2.0 * nnz * cfg.N / (ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (largest mean stage among kernels)
    peaks = ctx["peaks"]
    kern = {op: stage_ms[STAGE_OF_OP[op]] for op in sh.OPS if info["op_rows"][op] > 0}
    dom = max(kern, key=kern.get) if kern else "local"
    dom_ms = max(kern.get(dom, 0.0), 1e-9)
    ab = op_bytes(info, cfg.N, dom)
    ab_all = torch.tensor([float(ab)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ab_all, op=dist.ReduceOp.MAX)
    achieved = float(ab_all.item()) / (dom_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
            "traffic": traffic_from_profiles(cfg_name, world, dom),
            "algorithmic_bytes": int(ab_all.item()), "launch_ms": round(dom_ms, 5),
            "peak_source": peaks["source"],
            "gather_bytes": int(4 * cfg.N * info["op_nnz"][dom]) if dom != "pack" else None,
            "timing": "per-stage CUDA events on the launching stream, mean over the K "
                      "attribution steps, max over ranks"}
    fp32 = ctx["probes"]["fp32_tflops"]
    flops_dom = 2.0 * cfg.N * info["op_nnz"][dom]
    roof["fp32_frac"] = round(flops_dom / (dom_ms * 1e-3) / 1e12 / fp32, 4)

    # gather-aware term: the dominant local op's own column stream through the
    # pure gather probe, plus uniform-random gathers from L2- and HBM-resident
    # tables
    gather = None
    if world == 1 and primary or (world == 1 and args.gather_all):
        gather = gather_probes(sh, torch, dev, stream, Bd, col_l, lo, hi, cfg.N, flush)
        if gather and dom == "local":
            roof["gather_floor_ms"] = gather["csr_stream_ms"]
            roof["gather_frac"] = round(gather["csr_stream_ms"] / dom_ms, 4)
            # the row deliveries through L2 (one N*4-byte source row per
            # nonzero) against the measured random-row rate of an
            # L2-resident table: the bound of an L2-resident gather (c3)
            l2 = gather.get("l2_random_gbs")
            if l2:
                got = roof["gather_bytes"] / (dom_ms * 1e-3) / 1e9
                roof["l2_gather"] = {"achieved_gbs": round(got, 1), "peak_gbs": l2,
                                     "frac": round(got / l2, 4),
                                     "peak_source": "measured (gather_probe.l2_random_gbs)"}

    # ---- step-level roofline: T_roof = max over ranks of
    # max(HBM / BW_HBM, FLOP / FP32, NVLink / BW_NVL)
    nvl_bw = (ctx["nvlink"] or {}).get("ipc_store_gbs")
    per = []
    for tr in all_terms:
        hbm, flop, nvl, nnz_g, snd, rcv = tr.cpu().numpy().tolist()
        th = hbm / (peaks["hbm_gbs"] * 1e9)
        tf = flop / (fp32 * 1e12)
        tn = nvl / (nvl_bw * 1e9) if nvl_bw and nvl > 0 else 0.0
        per.append({"hbm_bytes": int(hbm), "flop": int(flop), "nvlink_bytes": int(nvl),
                    "nnz": int(nnz_g), "t_hbm_ms": th * 1e3, "t_fp32_ms": tf * 1e3,
                    "t_nvl_ms": tn * 1e3})
    t_roof = max(max(p["t_hbm_ms"], p["t_fp32_ms"], p["t_nvl_ms"]) for p in per)
    bound_of = lambda p: max((("hbm", p["t_hbm_ms"]), ("fp32", p["t_fp32_ms"]),
                              ("nvlink", p["t_nvl_ms"])), key=lambda x: x[1])[0]
    worst = max(per, key=lambda p: max(p["t_hbm_ms"], p["t_fp32_ms"], p["t_nvl_ms"]))
    nnz_r = [p["nnz"] for p in per]
    nvl_r = [p["nvlink_bytes"] for p in per]
    step_roof = {
        "t_roof_ms": round(t_roof, 5), "t_iter_ms": round(ms, 5),
        "frac": round(t_roof / ms, 4), "bound": bound_of(worst),
        "peaks": {"hbm_gbs": peaks["hbm_gbs"], "fp32_tflops": fp32, "nvlink_gbs": nvl_bw},
        "per_rank": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in p.items()}
                     for p in per],
        "imbalance_nnz_max_over_mean": round(max(nnz_r) / max(1e-9, np.mean(nnz_r)), 4),
        "imbalance_nvlink_max_over_mean": (round(max(nvl_r) / np.mean(nvl_r), 4)
                                           if world > 1 and np.mean(nvl_r) > 0 else None)}
    if gather:
        step_roof["t_gather_l2_ms"] = round(worst["nnz"] * 4 * cfg.N / (gather["l2_random_gbs"] * 1e9) * 1e3, 5)
        step_roof["t_gather_hbm_ms"] = round(worst["nnz"] * 4 * cfg.N / (gather["hbm_random_gbs"] * 1e9) * 1e3, 5)
    if ctx.get("t_floor_ms") is not None:
        step_roof["t_floor_ms"] = ctx["t_floor_ms"]

    # exchange (NVLink) achieved bandwidth, per rank max(send, recv) bytes
    xbytes = 4 * cfg.N * max(info["send_b_rows"] + info["send_c_rows"],
                             info["recv_b_rows"] + info["recv_c_rows"])
    xb = torch.tensor([float(xbytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(xb, op=dist.ReduceOp.MAX)
    exch = None
    if world > 1 and args.xchg == "nccl" and stage_ms["exchange"] > 0:
        gbs = xb.item() / (stage_ms["exchange"] * 1e-3) / 1e9
        exch = {"mode": "nccl grouped send/recv", "bytes_max_rank": int(xb.item()),
                "ms": round(stage_ms["exchange"], 5), "achieved_gbs": round(gbs, 1),
                "peak_gbs": nvl_bw, "frac": round(gbs / nvl_bw, 4) if nvl_bw else None}
    elif world > 1:
        # fused exchange: the rows cross NVLink inside the producer launch
        prod = stage_ms["partial"]
        gbs = xb.item() / (prod * 1e-3) / 1e9 if prod > 0 else None
        exch = {"mode": "fused p2p stores (CUDA IPC over NVLink), producer on a high-priority "
                        "stream concurrent with the local SpMM",
                "nvml_nvlink_tx_bytes_per_step": ((nvl1[0] - nvl0[0]) // args.steps)
                if nvl0 and nvl1 else None,
                "nvml_nvlink_rx_bytes_per_step": ((nvl1[1] - nvl0[1]) // args.steps)
                if nvl0 and nvl1 else None,
                "expected_send_bytes_this_rank": 4 * cfg.N * (info["send_b_rows"] + info["send_c_rows"]),
                "bytes_max_rank": int(xb.item()),
                "signal_ms": round(stage_ms["exchange"], 5), "producer_ms": round(prod, 5),
                "achieved_gbs_over_producer": round(gbs, 1) if gbs else None,
                "peak_gbs": nvl_bw, "frac": round(gbs / nvl_bw, 4) if gbs and nvl_bw else None}

    # N3: one value refresh of the plan (same values; collective), timed on
    # the host around the call (the refresh returns after the device update)
    barrier()
    t0 = time.perf_counter()
    plan.update_values(val_l, row_ptr=rp_l, col=col_l, stream=stream)
    t_ref = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ref, op=dist.ReduceOp.MAX)

    res = {
        "refresh_seconds": round(float(t_ref.item()), 4),
        "config": cfg, "value": value, "ms": ms, "nnz": nnz, "info": info, "roofline": roof,
        "roofline_step": step_roof, "gather": gather, "exchange": exch, "launches": launches,
        "stage_ms": stage_ms, "per_rank": per_rank, "step_ms": step_ms,
        "bytes": {"joint": info["g_joint_rows"] * 4 * cfg.N,
                  "oblivious_allgather": info["g_oblivious_rows"] * 4 * cfg.N,
                  "col_based": info["g_col_rows"] * 4 * cfg.N,
                  "row_based": info["g_row_rows"] * 4 * cfg.N,
                  "block": info["g_block_rows"] * 4 * cfg.N,
                  "joint_vs_oblivious": (info["g_joint_rows"] / info["g_oblivious_rows"])
                  if info["g_oblivious_rows"] else None,
                  "setup_bytes": info["g_setup_bytes"]},
    }
    if primary:
        res.update(plan=plan, Bd=Bd, B_p=B_p, M=M, row_ptr=row_ptr, col=col, val=val)
    else:
        plan.free()
    return res


def summary(r):
    cfg = r["config"]
    return {"workload": f"{cfg.name}: {cfg.desc}", "value": round(r["value"], 3), "unit": "GFLOP/s",
            "ms_per_step": round(r["ms"], 5), "roofline": r["roofline"],
            "roofline_step": r["roofline_step"], "exchange": r["exchange"],
            "stages_ms": {k: round(v, 5) for k, v in r["stage_ms"].items()},
            "bytes": r["bytes"], "plan_seconds": round(r["info"]["plan_seconds"], 3),
            "refresh_seconds": r["refresh_seconds"]}


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--also", default=None,
                    help="comma list of configs measured after the headline one "
                         "(default: c4 when the headline is c3; 'none' for none)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--group-size", type=int, default=1)
    ap.add_argument("--split-recv", action="store_true", help="SHIRO_F_SPLIT_RECV (K2 and K5 as two launches)")
    ap.add_argument("--colmax", action="store_true", help="SHIRO_F_COVER_COLMAX")
    ap.add_argument("--balance", action="store_true", help="SHIRO_F_COVER_BALANCE (R18)")
    ap.add_argument("--mode", default="joint", choices=["joint", "col", "row"])
    ap.add_argument("--xchg", default="p2p", choices=["p2p", "nccl"],
                    help="fused NVLink exchange (default) or NCCL grouped send/recv")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-probes", action="store_true", help="skip the NVLink / T_floor probes")
    ap.add_argument("--gather-all", action="store_true", help="gather probes for --also configs too")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    import shiro_gen
    cfg = shiro_gen.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return
    also = args.also if args.also is not None else ("c4" if args.config == "c3" else "none")
    also = [] if also in ("", "none") else [c for c in also.split(",") if c != args.config]

    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"       # keep stdout to the one JSON line
    import torch
    import torch.distributed as dist

    import paper_2512_20178_b200 as sh

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def fresh_id():
        """A new ncclUniqueId for each plan's communicator (ids are single-use)."""
        if world == 1:
            return None
        obj = [sh.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]
    # a dedicated (capturable) stream: shiro_spmm replays one CUDA graph per step
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    clocks = ClockSampler(local)
    clocks.start()
    probes = probe_peaks(sh, torch, dev, stream)
    pt = torch.tensor([probes["fp32_tflops"], probes["copy_gbs"]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(pt, op=dist.ReduceOp.MIN)
    probes["fp32_tflops"], probes["copy_gbs"] = [round(x, 2) for x in pt.cpu().numpy().tolist()]
    nvl = None
    if world > 1 and not args.no_probes:
        nvl = nvlink_probe(sh, torch, dist, dev, stream, world, rank, fresh_id())
    tfl = None
    if not args.no_probes:
        tfl = t_floor(sh, torch, dist, dev, stream, world, rank, fresh_id(), cfg.N, barrier)
    ctx = {"sh": sh, "torch": torch, "dist": dist, "world": world, "rank": rank, "dev": dev,
           "local": local,
           "stream": stream, "barrier": barrier, "fresh_id": fresh_id, "peaks": load_peaks(),
           "probes": probes, "nvlink": nvl, "t_floor_ms": tfl,
           "flush": torch.empty(256 << 20, dtype=torch.uint8, device=dev)}

    main_r = measure(args.config, args, ctx, primary=True)
    plan, Bd, B_p, M = main_r["plan"], main_r["Bd"], main_r["B_p"], main_r["M"]
    nnz = main_r["nnz"]

    # end to end through the public API with host buffers (pinned): every
    # step uploads its B_p and downloads its C_p inside the timed region.
    # shiro_spmm_host_batch pipelines the K steps (upload of step i overlaps
    # the download of step i-1); the single-call shiro_spmm_host time is
    # reported beside it.
    e2e = None
    if not args.no_e2e:
        Bhs = [torch.from_numpy(B_p).pin_memory() for _ in range(2)]
        Chs = [torch.empty((M, cfg.N)).pin_memory() for _ in range(2)]
        plan.spmm_host(Bhs[0], Chs[0], stream)
        plan.spmm_host_batch([Bhs[i % 2] for i in range(args.warmup)],
                             [Chs[i % 2] for i in range(args.warmup)], stream)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        plan.spmm_host_batch([Bhs[i % 2] for i in range(args.steps)],
                             [Chs[i % 2] for i in range(args.steps)], stream)
        tb = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64, device=dev)
        tt = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            plan.spmm_host(Bhs[0], Chs[0], stream)
            tt.append(time.perf_counter() - t0)
        te = torch.tensor(tt, dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        te_mean = float(te.mean().item())
        tb_step = float(tb.item())
        if not np.array_equal(Chs[(args.steps - 1) % 2][:4].numpy(), Chs[0][:4].numpy()):
            raise RuntimeError("e2e: batch and single-call results differ")
        e2e = {"value": round(2.0 * nnz * cfg.N / tb_step / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(B_p.nbytes) * world,
               "d2h_bytes_per_step": int(M * cfg.N * 4) * world,
               "ms_per_step": round(tb_step * 1e3, 4),
               "api": "shiro_spmm_host_batch (pipelined over the K steps)",
               "single_call_ms_per_step": round(te_mean * 1e3, 4),
               "single_call_value": round(2.0 * nnz * cfg.N / te_mean / 1e9, 3)}
    plan.free()
    launches = main_r["launches"]
    row_ptr, col, val = main_r["row_ptr"], main_r["col"], main_r["val"]
    for k in ("plan", "Bd", "B_p", "row_ptr", "col", "val"):
        main_r.pop(k, None)

    others = {}
    for c in also:
        others[c] = summary(measure(c, args, ctx, primary=False))

    clk = clocks.stop()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, row_ptr, col, val, shiro_gen.gen_B(cfg.seed, 0, cfg.n, cfg.N))

    if rank == 0:
        step_ms = main_r["step_ms"]
        out = {
            "metric": METRIC, "value": round(main_r["value"], 3), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(main_r["ms"], 5),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "n": cfg.n, "nnz": nnz, "N": cfg.N,
                       "P": world, "group_size": args.group_size,
                       "plan": ("split-recv " if args.split_recv else "") + args.mode +
                               (" col-max" if args.colmax else " row-max") +
                               (" balanced (R18)" if args.balance else ""),
                       "partition": "uniform 1D rows (larger blocks first)",
                       "l2": "flushed (256 MiB memset) before every timed step",
                       "exchange": (args.xchg if world > 1 else "none"),
                       "parallelism": f"1D row partition over {world} rank(s)"},
            "roofline": main_r["roofline"],
            "roofline_step": main_r["roofline_step"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "peaks_measured": {"fp32_tflops": probes["fp32_tflops"], "copy_gbs": probes["copy_gbs"],
                               "nvlink": nvl, "sms": probes["sms"],
                               "how": "FP32: 8 FMA chains/thread x 8 CTAs/SM; copy: float4 "
                                      "1 GiB (read+write bytes); min over ranks"},
            "bytes": main_r["bytes"],
            "bytes_table": bytes_table(),
            "exchange": main_r["exchange"],
            "gather_probe": main_r["gather"],
            "stages_ms": {k: round(v, 5) for k, v in main_r["stage_ms"].items()},
            "stages_ms_per_rank": main_r["per_rank"],
            "step_ms": {"median": round(float(np.median(step_ms)), 5),
                        "p10": round(float(np.percentile(step_ms, 10)), 5),
                        "p90": round(float(np.percentile(step_ms, 90)), 5)},
            "plan_seconds": round(main_r["info"]["plan_seconds"], 3),
            "refresh_seconds": main_r["refresh_seconds"],
            "also": others,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
