#!/bin/bash
# c5 (1.06 B nnz, N=64) at P=4 and P=2 on one 4-GPU box with the final code
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5m_build.log 2>&1
python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" > gpurun_out/c5m_gen.log 2>&1
for NG in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((NG-1))) timeout 1800 env ${C5ENV} python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG \
    --master-addr 127.0.0.1 --master-port 2951$NG bench.py --gpus $NG --config c5 --also none --no-e2e --steps 10 \
    > gpurun_out/c5m${TAG}_P$NG.json 2> /tmp/c5m_P$NG.err
  tail -c 2000 /tmp/c5m_P$NG.err > gpurun_out/c5m${TAG}_P$NG.errtail
done
echo done > gpurun_out/c5m_done.txt
