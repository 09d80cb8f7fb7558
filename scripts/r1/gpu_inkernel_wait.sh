# in-kernel READY wait of the remote SpMM (SHIRO_INKERNEL_WAIT): 2-process test + A/B at P=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/inkernel_wait.txt
: > $OUT
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x 2>&1 | tail -3 >> $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
SHIRO_INKERNEL_WAIT=1 SHIRO_P2P_TIMEOUT_MS=20000 timeout 300 $TR scripts/dist_check.py --config c2 --int >> $OUT 2>>gpurun_out/ikw_err.log || echo "FAILED dist_check" >> $OUT
for rep in 1 2; do
  for w in 1 0; do
    for c in c2 c4; do
      echo "== rep $rep $c SHIRO_INKERNEL_WAIT=$w" >> $OUT
      SHIRO_INKERNEL_WAIT=$w timeout 600 $TR bench.py --gpus 4 --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> $OUT 2>>gpurun_out/ikw_err.log || echo "FAILED rc=$?" >> $OUT
    done
  done
done
python - $OUT <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{"metric'):
        d=json.loads(l)
        print(d['config']['workload'][:3], 'ms',d['ms_per_step'], 'GF',round(d['value']), 'launches', d['gpu_launches'], 'median', d['step_ms']['median'])
    elif l.startswith('==') or l.startswith('{"config') or 'FAILED' in l or 'passed' in l or 'failed' in l:
        print(l.strip()[:300])
PY
