set -x
timeout 300 python tools/fused_check.py > gpurun_out/r02c_fused_check.log 2>&1; echo "exit=$?" >> gpurun_out/r02c_fused_check.log
BITSORT_KF_TRACE=1 timeout 300 python tools/fused_check.py --trace > gpurun_out/r02c_fused_trace.log 2>&1; echo "exit=$?" >> gpurun_out/r02c_fused_trace.log
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q --timeout 300 > gpurun_out/r02c_pytest_fused.log 2>&1; echo "exit=$?" >> gpurun_out/r02c_pytest_fused.log
echo done
