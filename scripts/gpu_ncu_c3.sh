#!/bin/bash
# ncu --set full of c3's k_spmm with the final kernel (8 rows per warp, HINT 1)
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n3_build.log 2>&1
python scripts/prof_one.py --config c3 > gpurun_out/n3_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 1 -c 1 -o /tmp/n3 python scripts/prof_one.py --config c3 > /tmp/n3_ncu.log 2>&1
ncu -i /tmp/n3.ncu-rep --page raw --csv > gpurun_out/n3_c3_raw.csv 2>&1
echo done > gpurun_out/n3_done.txt
