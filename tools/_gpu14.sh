RCP_MTTKRP_PATH=tiles timeout 600 python tools/lab/mttkrp_vs_oracle.py > gpurun_out/cmp_tiles.log 2>&1
export RCP_MTTKRP_PATH=tiles
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench14.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/t14.log
