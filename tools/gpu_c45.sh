timeout 600 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c45_c4_a.json 2>&1
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c45_c5_a.json 2>&1
timeout 900 python bench.py --config all --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c45_all.jsonl 2>&1
