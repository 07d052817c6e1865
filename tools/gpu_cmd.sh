set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --config all --steps 20 --warmup 3 > gpurun_out/bench_all_v7.jsonl 2> gpurun_out/bench_all_v7.err
timeout 300 python bench.py > gpurun_out/bench_default.json 2>&1 || exit 1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
for c in C2 C3 C4 C5; do python tools/run_one.py --config $c --iters 1 > /dev/null 2>&1 || exit 2; done
timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prof_c2_final -f python tools/run_one.py --config C2 --iters 1 > gpurun_out/ncu_full.log 2>&1
for c in C3 C4 C5; do timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_$c.csv python tools/run_one.py --config $c --iters 1 > /dev/null 2>&1; done
