cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_env_sweep.sh "c2:SHIRO_CHUNK=32 c2:SHIRO_CHUNK=64 c2:SHIRO_CHUNK=128 c4:SHIRO_CHUNK=128 c4:SHIRO_CHUNK=256 c4:SHIRO_CHUNK=512 c3:SHIRO_CHUNK=256 c3:SHIRO_CHUNK=512 c3:SHIRO_CHUNK=1024"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
