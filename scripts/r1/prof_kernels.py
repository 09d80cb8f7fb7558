"""One SpMM (P=1) and one gather probe over the same column stream, for ncu.

    python scripts/prof_kernels.py --config c2 [--reps 2]
"""
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
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
cfg = shiro_gen.CONFIGS[args.config]
rp, col, val = shiro_gen.gen_matrix(cfg, cache_dir=os.environ.get("SHIRO_GEN_CACHE", "/tmp/shiro_gen_cache"))
pl = sh.Plan.distributed(0, 1, cfg.n, np.array([0, cfg.n]), rp, col, val, cfg.N)
B = torch.from_numpy(shiro_gen.gen_B(cfg.seed, 0, cfg.n, cfg.N)).cuda()
C = torch.empty_like(B)
idx = torch.from_numpy(col.astype(np.int32)).cuda()
out = torch.empty(((idx.numel() + 255) // 256, cfg.N), device="cuda")
for _ in range(args.reps):
    pl.spmm(B, C)
    sh.probe_gather(B, idx, out, 256)
torch.cuda.synchronize()
print("ok", pl.info()["op_nnz"])
