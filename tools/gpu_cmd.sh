timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_scan.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_scan.log
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_small.json 2>>gpurun_out/c1.err
