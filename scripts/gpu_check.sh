cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for g in 1 0; do SHIRO_GRAPH=$g timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>gpurun_out/b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graph=$g', d['value'], d['ms_per_step'], d['stages_ms']['local'])"; done
tail -3 gpurun_out/b.err
