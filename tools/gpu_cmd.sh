timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "nccl or a2a or range_sort" > gpurun_out/pytest_a2a.log 2>&1; echo exit=$? >> gpurun_out/pytest_a2a.log
for c in C2 C4 C5; do
timeout 300 python bench.py --config $c --dist --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_dist_$c.json 2>&1
timeout 300 python bench.py --config $c --a2a --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_a2a_$c.json 2>&1
done
