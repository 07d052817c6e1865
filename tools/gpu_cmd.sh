timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "non_power" > gpurun_out/pytest_np2.log 2>&1; echo exit=$? >> gpurun_out/pytest_np2.log
