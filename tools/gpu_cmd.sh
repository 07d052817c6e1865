timeout 600 python tools/push_bench.py > gpurun_out/push_bench.jsonl 2> gpurun_out/push_bench.err
timeout 300 python bench.py --config C2 --push --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_push_1rank.json 2> gpurun_out/bench_push.err
timeout 300 python bench.py --config C2 --dist --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_rs_1rank.json 2>> gpurun_out/bench_push.err
