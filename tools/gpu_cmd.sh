timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "BUCKETED" > gpurun_out/pytest_quick.log 2>&1; echo quick_exit=$? >> gpurun_out/pytest_quick.log
if grep -q "quick_exit=0" gpurun_out/pytest_quick.log; then
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config all --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
for c in C4 C5; do BITSORT_NO_XWIDE=1 timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_noxw_$c.json 2>&1; done
fi
