python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
python tools/run_one.py --config C2 --iters 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"bucket_" -c 4 -o gpurun_out/prof_c2_final python tools/run_one.py --config C2 --iters 1 > gpurun_out/ncu_full.log 2>&1
for c in C3 C4 C5; do python tools/run_one.py --config $c --iters 1 > gpurun_out/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_$c.csv python tools/run_one.py --config $c --iters 1 > /dev/null 2>&1; done
