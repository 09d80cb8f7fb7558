"""LDG.128 register gathers vs TMA tile::gather4 shared-memory staging, as a
pure row-gather probe over the SpMM column streams of c2/c3/c4 and over
uniform random rows (L2-resident 32 MiB and HBM-resident 4 GiB tables).

    python scripts/tma_probe.py [--configs c2 c4 c3]

Prints one line per (stream, variant): ms per pass and delivered GB/s
(n_idx x 512 B / t); checks that every variant's sums agree bit for bit
(same summation order)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_20178_b200 as sh  # noqa: E402
import shiro_gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="*", default=["c2", "c4", "c3"])
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
N, CHUNK = 128, 256
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn):
    fn()
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(name, X, idx):
    idx = idx[: idx.numel() // 4 * 4]
    n = idx.numel()
    outs = {}
    variants = [("ldg", lambda o: sh.probe_gather(X, idx, o, CHUNK))]
    for st in (2, 4, 8):
        variants.append((f"tma_s{st}", lambda o, st=st: sh.probe_gather_tma(X, idx, o, CHUNK, st)))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for st in (8, 16, 24):      # warp-specialized ring, 4 CTAs x 8 warps per SM (round 2)
        variants.append((f"ws_s{st}", lambda o, st=st: sh.probe_gather_tma_ws(X, idx, o, st, 4 * sms)))
    for vname, fn in variants:
        rows = max((n + CHUNK - 1) // CHUNK, 4 * sms * 8)
        out = torch.zeros((rows, N), device="cuda")
        ms = timeit(lambda: fn(out))
        outs[vname] = out
        print(f"{name:28s} {vname:7s} {ms:8.4f} ms  {n * 4 * N / ms / 1e6:9.1f} GB/s", flush=True)
    ref = outs["ldg"]
    tot = float(ref.double().sum())
    for k, v in outs.items():
        if k.startswith("ws_"):        # different partial sums: compare totals
            t = float(v.double().sum())
            if abs(t - tot) > 1e-4 * abs(tot):
                print(f"  MISMATCH {k}: total {t:.6e} vs {tot:.6e}", flush=True)
        elif not torch.equal(v, ref):
            print(f"  MISMATCH {k}: max diff {float((v - ref).abs().max()):.3e}", flush=True)


for cfg in args.configs:
    c = shiro_gen.CONFIGS[cfg]
    rp, col, val = shiro_gen.gen_matrix(cfg, cache_dir=os.environ.get("SHIRO_GEN_CACHE", "/tmp/shiro_gen_cache"))
    X = torch.from_numpy(shiro_gen.gen_B(c.seed, 0, c.n, N)).cuda()
    run(f"{cfg} column stream", X, torch.from_numpy(col.astype(np.int32)).cuda())
    del X
g = torch.Generator(device="cuda").manual_seed(1)
for label, rows in (("random, 32 MiB table", (32 << 20) // 512), ("random, 4 GiB table", (4 << 30) // 512)):
    X = torch.rand((rows, N), device="cuda")
    idx = torch.randint(0, rows, (16 << 20,), device="cuda", generator=g, dtype=torch.int32)
    run(label, X, idx)
    del X
