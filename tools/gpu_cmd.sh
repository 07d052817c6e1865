timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_c2_e2e.json 2> gpurun_out/bench_c2_e2e.err
