#!/bin/bash
# round-2 multi-GPU bench: P=1 default line, then P=NG over c2/c3/c4
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
NG=${NG:-2}
TAG=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
if [ "${SKIP_P1:-0}" != "1" ]; then
  timeout 1200 python bench.py ${P1_ARGS} > gpurun_out/${TAG}_P1.json 2> gpurun_out/${TAG}_P1.err
fi
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus $NG --config c2 --also c4,c3 --no-e2e ${PN_ARGS} \
  > gpurun_out/${TAG}_P${NG}.json 2> gpurun_out/${TAG}_P${NG}.err
echo done >> gpurun_out/${TAG}_P${NG}.err
