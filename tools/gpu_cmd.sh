timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_r$i.json 2>&1; done
