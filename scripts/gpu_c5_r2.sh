#!/bin/bash
# c5 (1.07 B nnz) on one B200 box: plan digests at P=2/4/8 vs the oracle (CPU,
# in the background), sampled GPU parity at P=1/2, and the P=1 bench line.
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache SHIRO_C5=1 OMP_NUM_THREADS=$(nproc)
OUT=gpurun_out/c5r2
free -g > ${OUT}_mem.txt; nproc >> ${OUT}_mem.txt
python -c "import __graft_entry__ as g; g.build()" > ${OUT}_build.log 2>&1
( time python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" ) > ${OUT}_gen.log 2>&1
( timeout 5400 python -m pytest tests/test_c5.py -q -k digests -p no:cacheprovider > ${OUT}_digests.log 2>&1; echo "rc=$?" >> ${OUT}_digests.log;
  cp profiles/bytes_table.json ${OUT}_bytes_table.json; BYTES_TABLE_OUT=${OUT}_bytes_table.json timeout 2400 python scripts/bytes_table.py c5 > ${OUT}_bytes_table.log 2>&1 ) &
DIG=$!
timeout 2400 python -m pytest tests/test_c5.py -q -k product -p no:cacheprovider > ${OUT}_product.log 2>&1; echo "rc=$?" >> ${OUT}_product.log
timeout 1800 python bench.py --config c5 --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > ${OUT}_bench_P1.json 2> ${OUT}_bench_P1.err
free -g >> ${OUT}_mem.txt
wait $DIG
echo done >> ${OUT}_mem.txt
