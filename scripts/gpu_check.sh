cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
SHIRO_KVAR=10 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
bash scripts/sweep.sh "c2 c4 c3" "SHIRO_KVAR=4;SHIRO_KVAR=10;SHIRO_KVAR=11;SHIRO_KVAR=12;SHIRO_KVAR=13;SHIRO_KVAR=14"
cat gpurun_out/sweep.txt
