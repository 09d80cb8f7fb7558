# usage: bash scripts/gpu_multi.sh P [configs]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-2}
CFGS=${2:-"c2 c4"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/multi_P$P.txt
: > $OUT
for a in "--config c1" "--config c2" "--config c2 --int --flags fused" "--config c2 --flags colmax" "--config c2 --flags nccl" "--config c2 --int --flags row"; do
  echo "== $a" >> $OUT
  SHIRO_P2P_TIMEOUT_MS=20000 timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
for c in $CFGS; do
  for x in p2p nccl; do
    echo "== bench $c $x" >> $OUT
    timeout 600 $TR bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --xchg $x >> $OUT 2>>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
  done
done
echo done
