cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-4}
export OMP_NUM_THREADS=$(nproc)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/step_P$P.txt
: > $OUT
for a in "--config c2 --int" "--config c2" "--config c4 --sample 3000" "--config c2 --int --flags colmax"; do
  echo "== $a" >> $OUT
  SHIRO_P2P_TIMEOUT_MS=20000 timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/step_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
for c in c2 c4 c3; do
  for fs in 1 0; do
    echo "== bench $c fused_step=$fs" >> $OUT
    SHIRO_FUSED_STEP=$fs timeout 600 $TR bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>>gpurun_out/step_err_P$P.log || echo "FAILED rc=$?" >> $OUT
  done
done
python scripts/show_multi.py $OUT
