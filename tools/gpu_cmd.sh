timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for c in C3 C2; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${c}_rep.json 2>&1; done
BITSORT_SLAB=0 timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_packed.json 2>&1
