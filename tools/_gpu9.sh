export RCP_MTTKRP_PATH=tiles
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off --log-file gpurun_out/launches9.csv python tools/prof_round.py > gpurun_out/ncu9.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_spmm -s 2 -c 1 -o gpurun_out/tile_spmm9 python tools/prof_round.py > gpurun_out/ncu9b.log 2>&1
