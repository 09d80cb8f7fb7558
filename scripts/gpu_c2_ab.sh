#!/bin/bash
# c2 at P = 4 / 2: rows in flight (SHIRO_U128=4) and L2 policy (SHIRO_L2HINT=0) A/B, twice.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2ab_build.log 2>&1
OUT=gpurun_out/c2ab.txt; : > $OUT
for NG in 4 2; do
  if [ $NG = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; fi
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
  for rep in 1 2; do
    for e in X=0 SHIRO_U128=4 SHIRO_L2HINT=0 "SHIRO_U128=4 SHIRO_L2HINT=0"; do
      env $e timeout 600 $TR bench.py --gpus $NG --config c2 --also none --no-e2e --no-probes --no-cpu-baseline > /tmp/m.json 2>/tmp/m.err
      python - "$NG" "$e" >> $OUT <<'PY'
import json,sys
try:
    d=[json.loads(l) for l in open('/tmp/m.json') if l.strip().startswith('{')][-1]
    print('P', sys.argv[1], sys.argv[2], 'ms', d['ms_per_step'], 'median', d['step_ms']['median'], d['stages_ms'])
except Exception as e: print('P', sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/m.err').read()[-300:])
PY
    done
  done
  unset CUDA_VISIBLE_DEVICES
done
echo done >> $OUT
