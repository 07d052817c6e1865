timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "DIRECT or emulated or nccl or BUCKETED" > gpurun_out/pytest_quick.log 2>&1; echo quick_exit=$? >> gpurun_out/pytest_quick.log
if grep -q "quick_exit=0" gpurun_out/pytest_quick.log; then
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for c in C1 C2 C4; do timeout 300 python bench.py --config $c --path DIRECT --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_direct_$c.json 2>&1; done
for c in C2 C4 C5; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --dist --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_dist_$c.json 2> gpurun_out/bench_dist_$c.err; done
fi
