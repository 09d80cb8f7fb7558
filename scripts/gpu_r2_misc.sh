#!/bin/bash
# round-2 misc on one B200: warp-specialized TMA probe check + full probe, c4 hot-mark A/B
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1
timeout 120 python scripts/tma_ws_check.py > gpurun_out/m_tma_ws_check.txt 2>&1; echo "rc=$?" >> gpurun_out/m_tma_ws_check.txt
if grep -q MISMATCH gpurun_out/m_tma_ws_check.txt || ! grep -q "rc=0" gpurun_out/m_tma_ws_check.txt; then
  echo "skip full probe" >> gpurun_out/m_tma_ws_check.txt
else
  timeout 1200 python scripts/tma_probe.py --configs c2 c4 c3 > gpurun_out/m_tma_probe.txt 2>&1
fi
OUT=gpurun_out/m_hot_ab.txt; : > $OUT
for rep in 1 2; do
for h in 0 48 64 96 128; do
  SHIRO_HOT_MB=$h timeout 600 python bench.py --config c4 --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-probes > /tmp/b.json 2>/tmp/b.err
  python -c "
import json; d=json.load(open('/tmp/b.json')); print('c4 hot_mb=$h', 'ms', d['ms_per_step'], 'kernel', d['roofline']['launch_ms'], 'gather_frac', d['roofline'].get('gather_frac'))" >> $OUT 2>&1 || tail -3 /tmp/b.err >> $OUT
done
done
echo done > gpurun_out/m_done.txt
