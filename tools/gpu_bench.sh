python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "exit=$?" >> gpurun_out/bench_c2.err
python bench.py --config all --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err; echo "exit=$?" >> gpurun_out/bench_all.err
python bench.py --config C2 --path DIRECT --steps 50 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c2_direct.json 2>&1
