#!/bin/bash
# A/B of the N=128 rows-in-flight change on NG GPUs (default U=8 vs SHIRO_U128=4)
# plus the multi-GPU exactness tests.
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
NG=${NG:-2}
T=gpurun_out/ab${NG}
python -c "import __graft_entry__ as g; g.build()" > ${T}_build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_multigpu.py -q -p no:cacheprovider > ${T}_mgtests.log 2>&1; echo "rc=$?" >> ${T}_mgtests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
OUT=${T}_sweep.txt; : > $OUT
run() {  # config, also, env...
  local c=$1; local al=$2; shift; shift
  env "$@" timeout 1200 $TR bench.py --gpus $NG --config $c --also $al --no-e2e --no-probes --no-cpu-baseline > /tmp/m.json 2>/tmp/m.err
  python - "$c" "$*" >> $OUT <<'PY'
import json,sys
try:
    for line in open('/tmp/m.json'):
        line=line.strip()
        if not line.startswith('{'): continue
        d=json.loads(line); print(sys.argv[1], sys.argv[2], 'ms', d['ms_per_step'], 'GF', d['value'], 'frac', d['roofline'].get('frac'), 'also', {k: (v.get('ms_per_step'), v.get('value')) for k, v in (d.get('also') or {}).items()})
except Exception as e: print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/m.err').read()[-600:])
PY
}
for rep in 1 2; do
  run c3 c4 X=0
  run c3 c4 SHIRO_U128=4
  run c2 none X=0
  run c2 none SHIRO_U128=4
done
echo done >> $OUT
