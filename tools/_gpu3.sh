timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/t3.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.log 2>&1
RCP_MTTKRP_PATH=rows timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench3_rows.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off --log-file gpurun_out/launches3.csv python tools/prof_round.py > gpurun_out/ncu3.log 2>&1
