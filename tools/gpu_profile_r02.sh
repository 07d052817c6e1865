# Round-2 measurement refresh (run through gpurun from the repo root): bench
# lines, reference arm, ncu launch list, ncu full captures (C2 KB3/KB4 and the
# fused KF ring kernel), DRAM traffic per kernel for C1-C5.
set -x
timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 1500 python bench.py --config all --steps 20 --warmup 3 > gpurun_out/r02_bench_all.jsonl 2> gpurun_out/r02_bench_all.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r02_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bucket_ -c 2 -f -o gpurun_out/r02_prof_c2 \
    python tools/run_one.py --config C2 --iters 1 > gpurun_out/r02_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -c 1 -f -o gpurun_out/r02_prof_kf_c2 \
    python tools/run_one.py --config C2 --path FUSED --iters 1 > gpurun_out/r02_ncu_kf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_sort -c 1 -f -o gpurun_out/r02_prof_ks_c1 \
    python tools/run_one.py --config C1 --path SMALL --iters 1 > gpurun_out/r02_ncu_ks.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/r02_bench_c1_ks.json 2> gpurun_out/r02_bench_c1_ks.err
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/r02_bench_c4_chunked.json 2> gpurun_out/r02_bench_c4.err
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/r02_bench_c5_chunked.json 2> gpurun_out/r02_bench_c5.err
timeout 300 python tools/width_bench.py > gpurun_out/r02_width_bench.jsonl 2>&1
for c in C1 C2 C3 C4 C5; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -c 10 --csv \
      --log-file gpurun_out/r02_traffic_$c.csv python tools/run_one.py --config $c --path AUTO --iters 1 > gpurun_out/r02_traffic_$c.log 2>&1
done
echo done > gpurun_out/r02_profile.done
