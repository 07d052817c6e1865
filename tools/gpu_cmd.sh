BITSORT_TMA_SINGLE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C2 or slab or non_power or BUCKETED" > gpurun_out/pytest_single.log 2>&1; echo exit=$? >> gpurun_out/pytest_single.log
for v in "" "BITSORT_TMA_SINGLE=1"; do env $v timeout 300 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > "gpurun_out/bench_C2_$v.json" 2>&1; done
