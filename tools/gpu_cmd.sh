timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config C1 --path DIRECT --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c1.json 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2_default.json 2> gpurun_out/bench_c2_default.err
