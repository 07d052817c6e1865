timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "more_than" > gpurun_out/pytest_big.log 2>&1; echo exit=$? >> gpurun_out/pytest_big.log
