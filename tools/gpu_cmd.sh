timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or slab or non_power or BUCKETED or signed" > gpurun_out/pytest_q.log 2>&1; echo exit=$? >> gpurun_out/pytest_q.log
for i in 1 2; do timeout 300 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_r$i.json 2>&1; done
