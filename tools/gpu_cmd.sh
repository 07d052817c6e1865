timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for c in C2 C3 C1; do timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${c}_dr.json 2>&1; done
