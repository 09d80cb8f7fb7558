"""Sanity check of the warp-specialized TMA gather probe on a small input
(run under `timeout`): totals must match the LDG probe."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_20178_b200 as sh  # noqa: E402

X = torch.rand((1 << 14, 128), device="cuda")
idx = torch.randint(0, 1 << 14, (1 << 16,), device="cuda", dtype=torch.int32)
ref = torch.zeros((256, 128), device="cuda")
sh.probe_gather(X, idx, ref, 256)
for st in (8, 16, 24):
    for ctas in (1, 4, 148 * 4):
        out = torch.zeros((ctas * 8, 128), device="cuda")
        sh.probe_gather_tma_ws(X, idx, out, st, ctas)
        torch.cuda.synchronize()
        a, b = float(out.double().sum()), float(ref.double().sum())
        print(st, ctas, a, b, "OK" if abs(a - b) <= 1e-5 * abs(b) else "MISMATCH", flush=True)
