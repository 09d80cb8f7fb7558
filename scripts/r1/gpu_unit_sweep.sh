# unit-size rule sweep: c2 at P = 4, 2, 1 plus c3/c4 at P = 1 (run with gpurun --gpus 4)
cd $GRAFT_REPO_ROOT
S4="c2:SHIRO_WAVES=4 c2:SHIRO_WAVES=2 c2:SHIRO_WAVES=8 c2:SHIRO_WAVES=4,SHIRO_CHUNK_MIN=16 c2:SHIRO_WAVES=4,SHIRO_CHUNK_MIN=32 c2:SHIRO_WAVES=4,SHIRO_HUB_MIN=256 c2:SHIRO_CHUNK=64"
bash scripts/gpu_env_sweep.sh "$S4" 4
bash scripts/gpu_env_sweep.sh "$S4" 2
bash scripts/gpu_env_sweep.sh "$S4 c4:SHIRO_WAVES=4 c3:SHIRO_WAVES=4 c4:SHIRO_WAVES=4,SHIRO_HUB_MIN=256" 1
