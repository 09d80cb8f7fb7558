cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c2}
CMD="python scripts/prof_kernels.py --config $CFG --reps 2"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm|k_probe" -s 2 -c 2 -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu.log 2>&1
echo done
