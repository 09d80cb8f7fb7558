# balanced cover (SHIRO_F_COVER_BALANCE, R18): parity + A/B bench at P=2 and P=4 (gpurun --gpus 4)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/balance.txt
: > $OUT
for P in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
  for a in "--config c3 --sample 2000 --flags balance" "--config c2 --int --flags balance"; do
    echo "== P=$P dist_check $a" >> $OUT
    SHIRO_P2P_TIMEOUT_MS=20000 timeout 600 $TR scripts/dist_check.py $a >> $OUT 2>>gpurun_out/balance_err.log || echo "FAILED rc=$?" >> $OUT
  done
  for b in "--balance" ""; do
    for c in c3 c4; do
      [ "$c" = c4 ] && [ "$P" = 2 ] && continue
      echo "== P=$P bench $c $b" >> $OUT
      timeout 600 $TR bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $b >> $OUT 2>>gpurun_out/balance_err.log || echo "FAILED rc=$?" >> $OUT
    done
  done
done
python - $OUT <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{"metric'):
        d=json.loads(l)
        print(d['config']['workload'][:3], d['config']['plan'], 'ms',d['ms_per_step'], 'GF',round(d['value']), 'bytes', d['bytes']['joint'], [round(r.get('local',0),3) for r in d['stages_ms_per_rank']])
    elif l.startswith('==') or l.startswith('{"config') or 'FAILED' in l:
        print(l.strip()[:300])
PY
