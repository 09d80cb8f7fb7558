#!/bin/bash
# round-2 multi-GPU: multi-GPU tests, P=NG benches over c2/c3/c4 (+ c5), P=1 line optional
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
NG=${NG:-2}
TAG=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_multigpu.py -q > gpurun_out/${TAG}_mgtests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_mgtests.log
if [ "${SKIP_P1:-1}" != "1" ]; then
  timeout 1200 python bench.py ${P1_ARGS} > gpurun_out/${TAG}_P1.json 2> gpurun_out/${TAG}_P1.err
fi
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
timeout 1800 $TR bench.py --gpus $NG --config c2 --also c4,c3 --no-e2e ${PN_ARGS} \
  > gpurun_out/${TAG}_P${NG}.json 2> gpurun_out/${TAG}_P${NG}.err
for v in ${VARIANTS}; do   # e.g. "SHIRO_INKERNEL_WAIT=0"
  env $v timeout 1800 $TR bench.py --gpus $NG --config c2 --also c4,c3 --no-e2e --no-probes ${PN_ARGS} \
    > gpurun_out/${TAG}_P${NG}_$v.json 2> gpurun_out/${TAG}_P${NG}_$v.err
done
if [ "${C5:-0}" = "1" ]; then
  # generate once in one process (cached): a rank generating c5 inside the
  # bench would hold the others at a barrier past NCCL's 10-minute timeout
  ( time python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" ) > gpurun_out/${TAG}_c5gen.log 2>&1
  timeout 2400 $TR bench.py --gpus $NG --config c5 --also none --no-e2e --no-probes --steps 10 \
    > gpurun_out/${TAG}_P${NG}_c5.json 2> gpurun_out/${TAG}_P${NG}_c5.err
fi
tail -c 3000 gpurun_out/${TAG}_P${NG}.err > gpurun_out/${TAG}_P${NG}.errtail; rm -f gpurun_out/${TAG}_P${NG}.err
echo done > gpurun_out/${TAG}_done.txt
