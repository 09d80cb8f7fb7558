cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
for c in c3 c4; do timeout 600 $TR bench.py --gpus 2 --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pr_$c.json 2>>gpurun_out/pr_err.log; done
bash scripts/gpu_prof_bench.sh c2
