#!/bin/bash
# Compact hot buffer (SHIRO_HOTBUF_MB) at P=1: exactness, c4 / c3 / c5 step
# times, ncu DRAM bytes of c4's k_spmm with and without it.
mkdir -p gpurun_out
export SHIRO_GEN_CACHE=/tmp/shiro_gen_cache SHIRO_C5=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/hb_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -p no:cacheprovider > gpurun_out/hb_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/hb_pytest.log
OUT=gpurun_out/hb_sweep.txt; : > $OUT
run() {  # config, env...
  local c=$1; shift
  env "$@" timeout 900 python bench.py --config $c --also none --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-probes > /tmp/b.json 2>/tmp/b.err
  python - "$c" "$*" >> $OUT <<'PY'
import json,sys
try:
    d=json.load(open('/tmp/b.json')); print(sys.argv[1], sys.argv[2], 'ms', d['ms_per_step'], 'GF', d['value'], 'frac', d['roofline']['frac'], 'gather_frac', d['roofline'].get('gather_frac'), 'launches', d.get('gpu_launches'))
except Exception as e: print(sys.argv[1], sys.argv[2], 'FAILED', e, open('/tmp/b.err').read()[-400:])
PY
}
for rep in 1 2; do
  for c in c2 c4 c3; do
    run $c X=0
    run $c SHIRO_U128=4
    run $c SHIRO_L2HINT=1
    run $c SHIRO_HOTBUF_MB=64
    run $c SHIRO_HOTBUF_MB=64 SHIRO_HOTBUF_POL=0
  done
done
for c in c4 c3; do
  for h in 32 96; do run $c SHIRO_HOTBUF_MB=$h; done
  run $c SHIRO_HOTBUF_MB=64 SHIRO_HOTBUF_POL=0 SHIRO_HOTBUF_WIN=1 SHIRO_PERSIST_MB=64 SHIRO_GRAPH=0
  run $c SHIRO_HOTBUF_MB=64 SHIRO_HOTBUF_POL=1 SHIRO_HOTBUF_WIN=1 SHIRO_PERSIST_MB=64 SHIRO_GRAPH=0
  run $c SHIRO_GRAPH=0
done
for tag in base hb64; do
  if [ $tag = hb64 ]; then export SHIRO_HOTBUF_MB=64; else unset SHIRO_HOTBUF_MB; fi
  python scripts/prof_one.py --config c4 > gpurun_out/hb_plain_$tag.log 2>&1 && \
    ncu --set full --clock-control none -k regex:k_spmm -s 1 -c 1 -o /tmp/hb_$tag python scripts/prof_one.py --config c4 > /tmp/hb_ncu_$tag.log 2>&1
  ncu -i /tmp/hb_$tag.ncu-rep --page raw --csv > gpurun_out/hb_c4_${tag}_raw.csv 2>&1
done
unset SHIRO_HOTBUF_MB
python -c "import shiro_gen; shiro_gen.gen_matrix('c5', cache_dir='/tmp/shiro_gen_cache')" > gpurun_out/hb_gen.log 2>&1
run c5 X=0
run c5 SHIRO_L2HINT=1
run c5 SHIRO_HOTBUF_MB=64
run c5 SHIRO_HOTBUF_MB=96 SHIRO_HOTBUF_POL=0
echo done >> $OUT
