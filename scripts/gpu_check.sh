cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
bash scripts/sweep.sh "c2 c4 c3" "SHIRO_KVAR=4;SHIRO_KVAR=3"
cat gpurun_out/sweep.txt
