set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x -k "rank_above_64" 2>&1 | tail -30 > gpurun_out/t_r64.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -60 > gpurun_out/t_all.log
SEEDS=3 timeout 900 python tools/stress_rank.py > gpurun_out/stress.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_engine.py -q -x -k "rank_above_64 and sts-70" > gpurun_out/memcheck.log 2>&1
tail -5 gpurun_out/memcheck.log
timeout 1500 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_engine.py -q -x -k "rank_above_64 and sts-70" > gpurun_out/initcheck.log 2>&1
tail -5 gpurun_out/initcheck.log
