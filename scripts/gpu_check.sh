cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
bash scripts/sweep.sh "c2" "SHIRO_CHUNK=32;SHIRO_CHUNK=64;SHIRO_CHUNK=96;SHIRO_CHUNK=128;SHIRO_CHUNK=192;SHIRO_KVAR=3;SHIRO_KVAR=2"
cat gpurun_out/sweep.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_default.json 2>gpurun_out/b.err; python -c "import json; d=json.load(open('gpurun_out/bench_c2_default.json')); print(d['value'], d['clocks'], d['cpu_baseline']['value'], d['e2e'])"
