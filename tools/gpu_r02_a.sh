set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 1500 python bench.py --config all --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_all.jsonl 2> gpurun_out/r02_bench_all.err
echo done
