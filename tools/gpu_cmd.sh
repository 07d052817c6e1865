python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
python bench.py --config all --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
