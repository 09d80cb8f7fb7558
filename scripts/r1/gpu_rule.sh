cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-4}
export OMP_NUM_THREADS=$(nproc)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29511"
for c in c2 c3 c4; do
  ABLATION_ONLY=joint,joint-colmax timeout 1500 $TR scripts/ablation.py --config $c --group-size 1 --out gpurun_out/rule_${c}_P$P > gpurun_out/rule_${c}_P$P.log 2>&1
done
grep -h strategy gpurun_out/rule_*_P$P.log | cut -c1-200
