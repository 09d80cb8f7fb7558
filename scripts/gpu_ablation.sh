cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-4}
export OMP_NUM_THREADS=$(nproc)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
for c in ${2:-c4 c2}; do
  timeout 1500 $TR scripts/ablation.py --config $c --group-size 2 --out gpurun_out/ablation_${c}_P$P > gpurun_out/ablation_${c}_P$P.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
grep strategy gpurun_out/ablation_*_P$P.log
