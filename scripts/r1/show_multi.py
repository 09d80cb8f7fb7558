import json, sys
for l in open(sys.argv[1]):
    l = l.strip()
    if l.startswith("NCCL"):
        continue
    if l.startswith("{"):
        d = json.loads(l)
        if "metric" in d:
            print(" ", d["value"], d["ms_per_step"], {k: v for k, v in d["stages_ms"].items() if v}, "bytes/obl", round(d["bytes"]["joint_vs_oblivious"] or 0, 3))
        else:
            print(" ", {k: d[k] for k in ("lists_bit_exact", "bad_elements", "checked_rows", "max_abs_err")})
    else:
        print(l)
