#!/bin/bash
# Rows in flight per warp (SHIRO_U2=2: 16 float2 / 8 float4 gathers per batch,
# weights shuffled at use) and stream-only evict_first (SHIRO_L2HINT=1) at P=1.
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache SHIRO_C5=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u2_build.log 2>&1
OUT=gpurun_out/u2_sweep.txt; : > $OUT
run() {  # config, env...
  local c=$1; shift
  env "$@" timeout 900 python bench.py --config $c --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-probes > /tmp/b.json 2>/tmp/b.err
  python - "$c" "$*" >> $OUT <<'PY'
import json,sys
try:
    d=json.load(open('/tmp/b.json')); print(sys.argv[1], sys.argv[2], 'ms', d['ms_per_step'], 'GF', d['value'], 'frac', d['roofline']['frac'], 'gather_frac', d['roofline'].get('gather_frac'))
except Exception as e: print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/b.err').read()[-400:])
PY
}
for rep in 1 2; do
  for c in c2 c4 c3; do
    run $c X=0
    run $c SHIRO_U2=2
    run $c SHIRO_L2HINT=1
    run $c SHIRO_U2=2 SHIRO_L2HINT=1
  done
done
python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" > gpurun_out/u2_gen.log 2>&1
run c5 X=0
run c5 SHIRO_U2=2
run c5 SHIRO_L2HINT=1
run c5 SHIRO_U2=2 SHIRO_L2HINT=1
echo done >> $OUT
