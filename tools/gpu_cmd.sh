timeout 900 python tools/bench_ladder.py --out gpurun_out/r01_gpu_ladder > gpurun_out/ladder.log 2>&1; echo exit=$? >> gpurun_out/ladder.log
