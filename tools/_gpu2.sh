RCP_POISON=1 timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/t_poison.log
for i in 1 2 3 4 5; do RCP_POISON=1 timeout 600 python -m pytest tests/test_gpu_engine.py -m gpu -q -x -k rank_above_64 2>&1 | tail -3; done > gpurun_out/t_r64_loop.log
CFG=c3 SAMPLER=sts timeout 900 python tools/mttkrp_stats.py > gpurun_out/stats_c3.log 2>&1
CFG=c3 SAMPLER=arls-lev timeout 900 python tools/mttkrp_stats.py > gpurun_out/stats_c3a.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1
