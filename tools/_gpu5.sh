timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_spmm -s 2 -c 1 -o gpurun_out/tile_spmm python tools/prof_round.py > gpurun_out/ncu5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_scatter -s 2 -c 1 -o gpurun_out/pair_scatter python tools/prof_round.py >> gpurun_out/ncu5.log 2>&1
