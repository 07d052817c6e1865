timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo exit=$? >> gpurun_out/pytest_gpu.log
for v in "" "BITSORT_BUCKET_SHIFT=19" "BITSORT_BUCKET_SHIFT=18"; do env $v timeout 300 python bench.py --config C2 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_C2_$v.json 2>&1; done
