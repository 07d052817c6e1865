for c in C2 C3; do timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${c}_na.json 2>&1; done
