# launch list + full ncu capture of the dominant kernel for one bench config (N=1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c2}
timeout 900 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${CFG}_full.json 2> gpurun_out/bench_${CFG}_full.err
CMD="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_$CFG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
timeout 600 $CMD > gpurun_out/plain2_$CFG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/prof_${CFG}_full $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo done
# keep the report small enough to travel back: raw + source pages as CSV, rep compressed
if [ -f gpurun_out/prof_${CFG}_full.ncu-rep ]; then
  ncu -i gpurun_out/prof_${CFG}_full.ncu-rep --page raw --csv > gpurun_out/prof_${CFG}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_${CFG}_full.ncu-rep --page details --csv > gpurun_out/prof_${CFG}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_${CFG}_full.ncu-rep --page source --csv > gpurun_out/prof_${CFG}_source.csv 2>/dev/null
  xz -T0 -6 gpurun_out/prof_${CFG}_full.ncu-rep
  du -sh gpurun_out/prof_${CFG}_*
fi
rm -f gpurun_out/plain*.log
