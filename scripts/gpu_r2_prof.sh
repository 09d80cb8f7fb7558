#!/bin/bash
# round-2: GPU tests, default-bench launch list, ncu --set full of k_spmm
# (c3, c4, c4 hot marks) -- reports stay in /tmp, only CSV pages come back
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/p_smoke.log
if [ "${SKIP_PROF:-0}" = "1" ]; then echo done > gpurun_out/p_done.txt; exit 0; fi
timeout 900 python scripts/tma_probe.py --configs c2 c4 c3 > gpurun_out/p_tma_probe.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/p_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv $CMD > /tmp/p_ncu1.log 2>&1
for c in c3 c4; do
  python scripts/prof_one.py --config $c > gpurun_out/p_plain_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 -o /tmp/p_$c python scripts/prof_one.py --config $c > /tmp/p_ncu_$c.log 2>&1
  ncu -i /tmp/p_$c.ncu-rep --page raw --csv > gpurun_out/p_${c}_raw.csv 2>&1
  ncu -i /tmp/p_$c.ncu-rep --page details --csv > gpurun_out/p_${c}_details.csv 2>&1
done
SHIRO_HOT_MB=64 python scripts/prof_one.py --config c4 > gpurun_out/p_plain_c4hot.log 2>&1 && \
  SHIRO_HOT_MB=64 ncu --set full --clock-control none -k regex:k_spmm -s 1 -c 1 -o /tmp/p_c4hot python scripts/prof_one.py --config c4 > /tmp/p_ncu_c4hot.log 2>&1
ncu -i /tmp/p_c4hot.ncu-rep --page raw --csv > gpurun_out/p_c4hot_raw.csv 2>&1
du -sh gpurun_out > gpurun_out/p_du.txt
echo done > gpurun_out/p_done.txt
