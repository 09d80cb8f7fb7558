#!/bin/bash
# L2 policy sweep on c3 / c4 at P=1 (hot/cold marks, persisting set-aside, hints)
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2_build.log 2>&1
python -c "import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size, 'persist_max', getattr(p,'persisting_l2_cache_max_size',None))" > gpurun_out/l2_props.txt 2>&1
OUT=gpurun_out/l2_sweep.txt; : > $OUT
run() {  # config, env...
  local c=$1; shift
  env "$@" timeout 600 python bench.py --config $c --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-probes > /tmp/b.json 2>/tmp/b.err
  python - "$c" "$*" >> $OUT <<'PY'
import json,sys
try:
    d=json.load(open('/tmp/b.json')); print(sys.argv[1], sys.argv[2], 'ms', d['ms_per_step'], 'GF', d['value'], 'frac', d['roofline']['frac'], 'gather_frac', d['roofline'].get('gather_frac'))
except Exception as e: print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/b.err').read()[-400:])
PY
}
for c in c4 c3; do
  run $c X=0
  for h in 32 64 96; do run $c SHIRO_HOT_MB=$h; done
  for h in 32 64; do run $c SHIRO_HOT_MB=$h SHIRO_PERSIST_MB=$h; done
  run $c SHIRO_L2HINT=2
  run $c SHIRO_PREFETCH=1
  run $c SHIRO_PREFETCH=1 SHIRO_HOT_MB=64
  run $c SHIRO_PREFETCH=1 SHIRO_HOT_MB=32
done
run c2 X=0
run c2 SHIRO_PREFETCH=1
