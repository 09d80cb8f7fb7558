# usage: bash scripts/gpu_multi.sh P
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/multi_P$P.txt
: > $OUT
for a in "--config c1" "--config c1 --int" "--config c2" "--config c2 --int --flags fused" "--config c2 --flags colmax,nooverlap" "--config c2 --flags col" "--config c2 --flags row"; do
  echo "== $a" >> $OUT
  timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
for c in c2 c4; do
  echo "== bench $c" >> $OUT
  timeout 600 $TR bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-e2e >> $OUT 2>>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
echo done
