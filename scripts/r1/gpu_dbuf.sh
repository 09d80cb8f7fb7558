# usage: bash scripts/gpu_dbuf.sh P -- double-buffered fused exchange: parity + A/B bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/dbuf_P$P.txt
: > $OUT
for a in "--config c2" "--config c2 --int" "--config c2 --int --flags split" "--config c4 --sample 3000"; do
  echo "== $a" >> $OUT
  SHIRO_P2P_TIMEOUT_MS=20000 timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/dbuf_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
for c in c2 c4; do
  for db in 1 0; do
    echo "== bench $c SHIRO_DBUF=$db" >> $OUT
    SHIRO_DBUF=$db timeout 600 $TR bench.py --gpus $P --config $c --steps 20 --warmup 5 --no-cpu-baseline >> $OUT 2>>gpurun_out/dbuf_err_P$P.log || echo "FAILED rc=$?" >> $OUT
  done
done
python - $OUT <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{"metric'):
        d=json.loads(l)
        print(d['config']['workload'][:3], 'ms',d['ms_per_step'], 'GF',round(d['value']), 'launches', d['gpu_launches'], 'e2e', d['e2e']['value'] if d.get('e2e') else None, {k:round(v,4) for k,v in d['stages_ms'].items() if v})
    elif l.startswith('==') or l.startswith('{"config') or 'FAILED' in l:
        print(l.strip()[:300])
PY
