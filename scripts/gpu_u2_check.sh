#!/bin/bash
# Correctness of the current kernels (parity + multi-process modules, the
# two-phase consumer repeated), then the rows-in-flight / L2 hint sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u2c_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -q -x -m gpu -p no:cacheprovider > gpurun_out/u2c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/u2c_pytest.log
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -m gpu -k "two_process_fused" -p no:cacheprovider >> gpurun_out/u2c_cx_repeat.log 2>&1; echo "rep $i rc=$?" >> gpurun_out/u2c_cx_repeat.log
done
SHIRO_U2=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -p no:cacheprovider > gpurun_out/u2c_pytest_u2.log 2>&1; echo "rc=$?" >> gpurun_out/u2c_pytest_u2.log
bash scripts/gpu_u2_sweep.sh
