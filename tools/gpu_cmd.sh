timeout 300 python bench.py --config C2 --steps 50 --warmup 5 > gpurun_out/bench_C2_full.json 2>&1
BENCH_NO_KERNEL_TIMING=1 timeout 300 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_nokt.json 2>&1
