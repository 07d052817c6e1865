timeout 900 python bench.py --config all --steps 20 --warmup 3 > gpurun_out/bench_all_v9.jsonl 2> gpurun_out/bench_all_v9.err
timeout 300 python bench.py > gpurun_out/bench_default.json 2>&1
