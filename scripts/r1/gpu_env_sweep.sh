# usage: bash scripts/gpu_env_sweep.sh "c2:SHIRO_CHUNK=32 c2:SHIRO_CHUNK=64 c4:SHIRO_KERNEL=15" [P]
# one bench line per (config, env assignment); P>1 runs under torchrun
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${2:-1}
OUT=gpurun_out/env_sweep_P$P.txt
: > $OUT
for item in $1; do
  c=${item%%:*}; envs=${item#*:}
  if [ "$P" = 1 ]; then
    env ${envs//,/ } timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/es.json 2>>gpurun_out/es_err.log
  else
    env ${envs//,/ } timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/es.json 2>>gpurun_out/es_err.log
  fi
  python - "$item" gpurun_out/es.json >> $OUT <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    st={k: round(v,4) for k,v in d['stages_ms'].items() if v}
    print(f"{sys.argv[1]} ms={d['ms_per_step']:.4f} gflops={d['value']:.0f} stages={st} gather_frac={d['roofline'].get('gather_frac')}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
cat $OUT
