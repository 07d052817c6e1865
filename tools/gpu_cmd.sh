timeout 600 python tools/width_bench.py --cases u64_full > gpurun_out/width_bench4.jsonl 2> gpurun_out/width_bench4.err
timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_auto.json 2>>gpurun_out/c1.err
timeout 300 python bench.py --config C1 --path BUCKETED --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_bucketed.json 2>>gpurun_out/c1.err
BITSORT_SCAN=v1 timeout 300 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c1_v1.json 2>>gpurun_out/c1.err
