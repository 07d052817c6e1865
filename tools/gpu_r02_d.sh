set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1
timeout 600 python bench.py --config C1 > gpurun_out/r02d_bench_c1.json 2> gpurun_out/r02d_bench_c1.err
echo done
