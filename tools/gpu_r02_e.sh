set -x
timeout 900 python -m pytest tests/test_gpu_multiset.py tests/test_gpu_parity.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "exit=$?" >> gpurun_out/r02e_pytest.log
timeout 300 python tools/width_bench.py > gpurun_out/r02e_width_bench.jsonl 2> gpurun_out/r02e_width_bench.err
echo done
