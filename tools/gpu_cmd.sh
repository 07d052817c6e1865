timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
