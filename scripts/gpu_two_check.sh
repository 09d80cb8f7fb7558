#!/bin/bash
# Branch-free two-source row addressing: exactness (parity + multi-process
# modules) and c4 with the compact hot buffer (a two-source op) vs default.
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tc_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_hier.py tests/test_gpu_refresh.py -q -x -m gpu -p no:cacheprovider > gpurun_out/tc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tc_pytest.log
OUT=gpurun_out/tc_sweep.txt; : > $OUT
for e in X=0 SHIRO_HOTBUF_MB=64 X=0 SHIRO_HOTBUF_MB=64; do
  env $e timeout 600 python bench.py --config c4 --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-probes > /tmp/b.json 2>/tmp/b.err
  python -c "
import json,sys
d=json.load(open('/tmp/b.json')); print('c4', '$e', 'ms', d['ms_per_step'], 'GF', d['value'])" >> $OUT 2>&1
done
echo done >> $OUT
