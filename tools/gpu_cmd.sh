nproc; cat /proc/cpuinfo | grep "model name" | head -1; numactl -H 2>/dev/null | head -3
for t in 4 8 12 16; do BITSORT_COPY_THREADS=$t timeout 300 python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_copy_$t.json 2>&1; done
