set -x
timeout 300 python tools/fused_check.py > gpurun_out/r02b_fused_check.log 2>&1; echo "exit=$?" >> gpurun_out/r02b_fused_check.log
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q --timeout 300 > gpurun_out/r02b_pytest_fused.log 2>&1; echo "exit=$?" >> gpurun_out/r02b_pytest_fused.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/r02b_pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02b_pytest_gpu.log
echo done
