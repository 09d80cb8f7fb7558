#!/bin/bash
# c2 at P=NG: latency knobs of the small-op regime (unit waves, hub threshold, cover rule)
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
NG=${NG:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/k_c2_P${NG}.txt; : > $OUT
run() {   # label, env..., -- args
  local label=$1; shift
  local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 600 $TR bench.py --gpus $NG --config c2 --also none --no-e2e --no-probes --steps 30 "$@" > /tmp/k.json 2>/tmp/k.err
  python - "$label" >> $OUT <<'PY'
import json,sys
try:
    d=json.loads(open('/tmp/k.json').read().strip().split('\n')[-1])
    print(sys.argv[1], 'ms', d['ms_per_step'], 'median', d['step_ms']['median'], {k:round(v,4) for k,v in d['stages_ms'].items() if v})
except Exception as e: print(sys.argv[1], 'FAILED', e)
PY
}
run default X=0 --
run waves8 SHIRO_WAVES=8 --
run waves16 SHIRO_WAVES=16 --
run hub32 SHIRO_HUB_MIN=32 --
run hub16_waves8 SHIRO_HUB_MIN=16 SHIRO_WAVES=8 --
run colmax X=0 -- --colmax
run balance X=0 -- --balance
run perunit SHIRO_INKERNEL_WAIT=1 --
run nccl X=0 -- --xchg nccl
echo done >> $OUT
