timeout 600 python -m pytest tests/test_gpu_parity.py -k chunked -x -q --timeout 300 -p no:cacheprovider > gpurun_out/chk.log 2>&1; echo "exit=$?" >> gpurun_out/chk.log
