export RCP_MTTKRP_PATH=tiles
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/t6.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench6.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off --log-file gpurun_out/launches6.csv python tools/prof_round.py > gpurun_out/ncu6.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_spmm -s 2 -c 1 -o gpurun_out/tile_spmm6 python tools/prof_round.py > gpurun_out/ncu6b.log 2>&1
