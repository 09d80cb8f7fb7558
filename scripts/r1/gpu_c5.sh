# c5 (R-MAT scale 26) on P GPUs: sampled parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-4}
export OMP_NUM_THREADS=$(nproc)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
OUT=gpurun_out/c5_P$P.txt
: > $OUT
free -g >> $OUT
( time timeout 2400 $TR scripts/dist_check.py --config c5 --sample 2000 --no-lists ) >> $OUT 2> gpurun_out/c5_err_P$P.log
tail -5 gpurun_out/c5_err_P$P.log >> $OUT
timeout 2400 $TR bench.py --gpus $P --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline >> $OUT 2>> gpurun_out/c5_err_P$P.log
tail -3 gpurun_out/c5_err_P$P.log
echo done
