RCP_MTTKRP_PATH=tiles timeout 600 python tools/lab/mttkrp_vs_oracle.py > gpurun_out/cmp_tiles16.log 2>&1
export RCP_MTTKRP_PATH=tiles
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench16.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off --log-file gpurun_out/launches16.csv python tools/prof_round.py > gpurun_out/ncu16.log 2>&1
