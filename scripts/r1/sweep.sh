# usage: bash scripts/sweep.sh "<configs>" "<env settings separated by ;>"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CONFIGS=${1:-"c2 c4"}
IFS=';' read -ra ENVS <<< "${2:-SHIRO_SPMM=sync;SHIRO_RING=16}"
for c in $CONFIGS; do
  for e in "${ENVS[@]}"; do
    r=$(env $e timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/sweep_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms'], d['roofline']['frac'])")
    echo "$c | $e | $r" >> gpurun_out/sweep.txt
  done
done
echo done
