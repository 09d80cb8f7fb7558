#!/bin/bash
# one B200: GPU tests after the N=32/64 lane change, c5/c1 P=1 A/B, TMA ws probe, hot-mark A/B
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c2_pytest.log
python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" > /dev/null 2>&1
timeout 1200 python bench.py --config c5 --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2_bench_c5.json 2> gpurun_out/c2_bench_c5.err
timeout 600 python bench.py --config c2 --also c3,c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2_bench_c234.json 2> gpurun_out/c2_bench_c234.err
bash scripts/gpu_r2_misc.sh
echo done > gpurun_out/c2_done.txt
