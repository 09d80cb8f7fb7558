#!/bin/bash
# End-of-round measurements on a 4-GPU box: the 1-GPU default bench line +
# launch list + reference arm, the multi-GPU exactness tests, and the P = 2 / 4
# bench lines (default, old kernel shape A/B, c2, balanced cover, hierarchical).
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
T=gpurun_out/last
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > ${T}_smi.txt; nproc >> ${T}_smi.txt
python -c "import __graft_entry__ as g; g.build()" > ${T}_build.log 2>&1
# ---- 1 GPU
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python bench.py > ${T}1_bench.json 2> ${T}1_bench.err
timeout 600 python bench.py --config c2 --also none > ${T}1_bench_c2.json 2> ${T}1_bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${T}1_reference.json 2> ${T}1_reference.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > ${T}1_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${T}1_launches.csv $CMD > /tmp/ncu_last.log 2>&1
unset CUDA_VISIBLE_DEVICES
# ---- multi-GPU
timeout 1800 python -m pytest tests/test_gpu_multigpu.py -q -p no:cacheprovider > ${T}_mgtests.log 2>&1; echo "rc=$?" >> ${T}_mgtests.log
for NG in 4 2; do
  if [ $NG = 2 ]; then export CUDA_VISIBLE_DEVICES=0,1; fi
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
  timeout 1800 $TR bench.py --gpus $NG > ${T}${NG}_bench.json 2> ${T}${NG}_bench.err
  timeout 1800 $TR bench.py --gpus $NG --config c2 --also none --no-e2e > ${T}${NG}_bench_c2.json 2> ${T}${NG}_bench_c2.err
  SHIRO_U128=4 SHIRO_L2HINT=0 timeout 1800 $TR bench.py --gpus $NG --no-e2e --no-probes --no-cpu-baseline > ${T}${NG}_bench_oldshape.json 2> ${T}${NG}_bench_oldshape.err
  timeout 1800 $TR bench.py --gpus $NG --config c3 --also none --no-e2e --no-probes --balance > ${T}${NG}_bench_c3_balance.json 2> ${T}${NG}_bench_c3_balance.err
  if [ $NG = 4 ]; then
    timeout 1800 $TR bench.py --gpus $NG --config c4 --also c3 --no-e2e --no-probes --group-size 2 > ${T}${NG}_bench_hier_g2.json 2> ${T}${NG}_bench_hier_g2.err
  fi
  unset CUDA_VISIBLE_DEVICES
done
for f in ${T}*.err; do tail -c 2000 $f > $f.tail; rm -f $f; done
echo done > ${T}_done.txt
