# usage: bash scripts/gpu_multi.sh P [configs] [group]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-2}
CFGS=${2:-"c2 c4"}
GS=${3:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/multi_P$P.txt
: > $OUT
for a in "--config c2" "--config c2 --int --flags split" "--config c2 --int --flags nccl" "--config c2 --int --group-size $GS" "--config c4 --sample 3000"; do
  echo "== $a" >> $OUT
  SHIRO_P2P_TIMEOUT_MS=20000 timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
for c in $CFGS; do
  for opt in "--xchg p2p" "--group-size $GS"; do
    echo "== bench $c $opt" >> $OUT
    timeout 600 $TR bench.py --gpus $P --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $opt >> $OUT 2>>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
  done
done
echo done
