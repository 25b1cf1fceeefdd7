RCP_MTTKRP_PATH=tiles timeout 600 python tools/lab/mttkrp_vs_oracle.py > gpurun_out/cmp_tiles.log 2>&1
timeout 600 python tools/lab/mttkrp_vs_oracle.py > gpurun_out/cmp_rows.log 2>&1
