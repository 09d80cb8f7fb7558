# usage: bash scripts/gpu_kernel_sweep.sh "1 2 3" "c2 c3 c4"  -- SpMM kernel variant sweep at P=1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARS=${1:-"1 2 3 4 5"}
CFGS=${2:-"c2 c3 c4"}
OUT=gpurun_out/kernel_sweep.txt
: > $OUT
for v in $VARS; do
  echo "== SHIRO_KERNEL=$v pytest" >> $OUT
  SHIRO_KERNEL=$v timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> $OUT
  for c in $CFGS; do
    SHIRO_KERNEL=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ks_${v}_$c.json 2>>gpurun_out/ks_err.log
    python - "$v" "$c" gpurun_out/ks_${v}_$c.json >> $OUT <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(f"K={sys.argv[1]} {sys.argv[2]} ms={d['ms_per_step']:.4f} local={d['stages_ms']['local']:.4f} gflops={d['value']:.0f} gather_frac={d['roofline'].get('gather_frac')}")
except Exception as e:
    print("K", sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done
cat $OUT
