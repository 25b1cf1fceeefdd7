export RCP_MTTKRP_PATH=tiles
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench12.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off --log-file gpurun_out/launches12.csv python tools/prof_round.py > gpurun_out/ncu12.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/t12.log
