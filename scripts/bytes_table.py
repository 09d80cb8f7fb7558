#!/usr/bin/env python
"""Communicated bytes per SpMM step for every config at P = 2/4/8 (plus the
hierarchical inter/intra split for g = 2, 4), from HOST-ONLY loopback plans
of the library (the same planner as shiro_plan; no GPU needed).  Writes
profiles/bytes_table.json, which bench.py attaches as "bytes_table".

    python scripts/bytes_table.py [c1 c2 c3 c4 c5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_20178_b200 as sh  # noqa: E402
import shiro_gen  # noqa: E402


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
    path = os.environ.get("BYTES_TABLE_OUT", os.path.join(ROOT, "profiles", "bytes_table.json"))
    table = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        c = shiro_gen.CONFIGS[name]
        t0 = time.time()
        rp, col, val = shiro_gen.gen_matrix(name, cache_dir=os.environ.get("SHIRO_GEN_CACHE"))
        print(name, "generated", round(time.time() - t0, 1), "s", flush=True)
        for P in (2, 4, 8):
            part = sh.uniform_partition(c.n, P)
            row = {}
            for g in ([1, 2, 4] if P >= 4 else [1, 2]):
                if P % g or g == P:
                    continue
                t0 = time.time()
                pl = sh.Plan.loopback(P, c.n, part, rp, col, val, c.N, group_size=g,
                                      flags=sh.F_HOST_ONLY)
                i = pl.info()
                rb = 4 * c.N
                if g == 1:
                    row.update(joint=i["g_joint_rows"] * rb, col=i["g_col_rows"] * rb,
                               row=i["g_row_rows"] * rb, block=i["g_block_rows"] * rb,
                               oblivious=i["g_oblivious_rows"] * rb,
                               joint_vs_oblivious=round(i["g_joint_rows"] / i["g_oblivious_rows"], 5),
                               joint_vs_col=round(i["g_joint_rows"] / max(1, i["g_col_rows"]), 5),
                               max_recv_rank=i["g_max_recv_rows"] * rb,
                               setup_bytes=i["g_setup_bytes"],
                               plan_seconds=round(time.time() - t0, 2))
                else:
                    row[f"hier_g{g}"] = {"inter": i["g_hier_inter_rows"] * rb,
                                         "intra": i["g_hier_intra_rows"] * rb,
                                         "flat_inter": i["g_flat_inter_rows"] * rb}
                pl.free()
            table[f"{name}/P{P}"] = row
            print(name, P, row, flush=True)
        json.dump(table, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
