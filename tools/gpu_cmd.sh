timeout 300 python bench.py --config C2 --path DIRECT --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2d.json 2>&1
timeout 300 python bench.py --config C4 --path DIRECT --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C4d.json 2>&1
