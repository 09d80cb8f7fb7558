#!/bin/bash
# round-2 final measurements on NG GPUs (NG=1: GPU tests, smoke, default bench + launch list;
# NG>1: multi-GPU tests, default bench, balanced cover, hierarchical g=2)
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
NG=${NG:-1}
T=gpurun_out/final${NG}
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > ${T}_smi.txt; nproc >> ${T}_smi.txt; free -g >> ${T}_smi.txt
python -c "import __graft_entry__ as g; g.build()" > ${T}_build.log 2>&1
if [ "$NG" = "1" ]; then
  timeout 3000 python -m pytest tests -m gpu -q > ${T}_pytest.log 2>&1; echo "rc=$?" >> ${T}_pytest.log
  python -c "import __graft_entry__ as g; g.smoke()" > ${T}_smoke.log 2>&1; echo "rc=$?" >> ${T}_smoke.log
  timeout 1200 python bench.py > ${T}_bench.json 2> ${T}_bench.err
  timeout 600 python bench.py --config c2 --also none > ${T}_bench_c2.json 2> ${T}_bench_c2.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${T}_reference.json 2> ${T}_reference.err
  timeout 120 python scripts/tma_ws_check.py > ${T}_tma_ws_check.txt 2>&1; echo "rc=$?" >> ${T}_tma_ws_check.txt
  if grep -q "rc=0" ${T}_tma_ws_check.txt && ! grep -q MISMATCH ${T}_tma_ws_check.txt; then
    timeout 1200 python scripts/tma_probe.py --configs c2 c4 c3 > ${T}_tma_probe.txt 2>&1
  fi
  CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
  $CMD > ${T}_plain.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${T}_launches.csv $CMD > /tmp/ncu_final.log 2>&1
else
  timeout 1800 python -m pytest tests/test_gpu_multigpu.py -q > ${T}_mgtests.log 2>&1; echo "rc=$?" >> ${T}_mgtests.log
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
  timeout 1800 $TR bench.py --gpus $NG > ${T}_bench.json 2> ${T}_bench.err
  timeout 1800 $TR bench.py --gpus $NG --config c2 --also c4 --no-e2e > ${T}_bench_c2.json 2> ${T}_bench_c2.err
  timeout 1800 $TR bench.py --gpus $NG --config c3 --also none --no-e2e --no-probes --balance > ${T}_bench_c3_balance.json 2> ${T}_bench_c3_balance.err
  timeout 1800 $TR bench.py --gpus $NG --config c4 --also c3 --no-e2e --no-probes --group-size 2 > ${T}_bench_hier_g2.json 2> ${T}_bench_hier_g2.err
  for f in ${T}_bench*.err; do tail -c 2000 $f > $f.tail; rm -f $f; done
fi
echo done > ${T}_done.txt
