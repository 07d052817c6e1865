timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --config C2 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_$i.json 2>&1; done
timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C3.json 2>&1
