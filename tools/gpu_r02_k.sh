timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiset.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/r02k_pytest.log 2>&1; echo "exit=$?" >> gpurun_out/r02k_pytest.log
timeout 900 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench_c5.json 2>&1
timeout 900 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench_c4.json 2>&1
