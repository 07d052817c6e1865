# fused modes: parity + C1 timing of KD vs K2+K3 (development check)
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/kd_pytest.log 2>&1; echo "exit=$?" >> gpurun_out/kd_pytest.log
timeout 300 python tools/fused_check.py > gpurun_out/kd_fused_check.log 2>&1
BITSORT_KF_TRACE=1 timeout 300 python tools/fused_check.py --trace > gpurun_out/kd_trace.log 2>&1
