#!/bin/bash
# round-2 verification on one B200: GPU tests, then quick benches per config
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
nproc >> gpurun_out/r2_smi.txt; free -g >> gpurun_out/r2_smi.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
for c in ${CONFIGS:-c2 c3 c4}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
     > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
done
