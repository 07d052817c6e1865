set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/hyb_parity.log 2>&1; echo exit=$? >> gpurun_out/hyb_parity.log
timeout 600 python tools/sweep_env.py BITSORT_HYBRID_KPT 0 4 5 6 7 8 10 -- --steps 20 --warmup 3 > gpurun_out/hyb_sweep.jsonl 2>&1
