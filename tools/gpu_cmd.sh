for sh in 18 19 20; do BITSORT_BUCKET_SHIFT=$sh python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_s$sh.json 2>&1; done
BITSORT_PART=narrow python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_narrow.json 2>&1
for sh in 19 20; do BITSORT_BUCKET_SHIFT=$sh python bench.py --config C3 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_s$sh.json 2>&1; done
