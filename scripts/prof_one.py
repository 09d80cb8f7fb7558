#!/usr/bin/env python
"""Minimal driver for ncu: P = 1 plan of one config, `--steps` shiro_spmm
calls on a capturable stream (graph replays).  Usage:
    python scripts/prof_one.py --config c4 --steps 3"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_20178_b200 as sh  # noqa: E402
import shiro_gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
c = shiro_gen.CONFIGS[a.config]
rp, col, val = shiro_gen.gen_matrix(a.config, cache_dir=os.environ.get("SHIRO_GEN_CACHE"))
pl = sh.Plan.distributed(0, 1, c.n, np.array([0, c.n]), rp, col, val, c.N)
s = torch.cuda.Stream()
B = torch.from_numpy(shiro_gen.gen_B(c.seed, 0, c.n, c.N)).cuda()
C = torch.empty_like(B)
for _ in range(a.steps):
    pl.spmm(B, C, s)
s.synchronize()
print("ok", a.config, float(C[:4].sum()))
