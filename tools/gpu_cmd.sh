for i in 1; do timeout 300 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_pf.json 2>&1; done
timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C3_pf.json 2>&1
