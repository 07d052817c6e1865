# Round measurement refresh (run through gpurun from the repo root):
# bench lines, reference arm, ncu launch list, ncu full capture of one C2
# sort, DRAM traffic per kernel for C3-C5. Summaries: tools/summarize_profiles.py.
V=${1:-v10}
timeout 1500 python bench.py --config all --steps 20 --warmup 3 > gpurun_out/bench_all_$V.jsonl 2> gpurun_out/bench_all_$V.err
timeout 400 python bench.py > gpurun_out/bench_c2_$V.json 2> gpurun_out/bench_c2_$V.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_$V.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bucket_ -c 2 -f -o gpurun_out/prof_c2_final \
    python tools/run_one.py --config C2 --iters 1 > gpurun_out/ncu_full.log 2>&1
for c in C3 C4 C5; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 10 --csv \
      --log-file gpurun_out/traffic_$c.csv python tools/run_one.py --config $c --iters 1 > gpurun_out/traffic_$c.log 2>&1
done
echo done > gpurun_out/profile_round.done
