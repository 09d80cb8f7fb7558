cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-2}
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
timeout 300 $TR scripts/nccl_probe.py > gpurun_out/nccl_probe.txt 2>&1
NCCL_DEBUG=INFO timeout 600 $TR bench.py --gpus $P --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_P$P.txt 2> gpurun_out/nccl_debug.txt
OUT=gpurun_out/multi_P$P.txt
: > $OUT
for a in "--config c2" "--config c2 --int --flags split" "--config c2 --flags colmax,nooverlap" "--config c2 --flags col" "--config c2 --flags row"; do
  echo "== $a" >> $OUT
  timeout 300 $TR scripts/dist_check.py $a >> $OUT 2>gpurun_out/multi_err_P$P.log || echo "FAILED rc=$?" >> $OUT
done
echo done
