set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/r02j_pytest_gpu.log 2>&1; echo "exit=$?" >> gpurun_out/r02j_pytest_gpu.log
timeout 900 python tools/fuzz_long.py --minutes 10 --seed 2027 > gpurun_out/r02j_fuzz.log 2>&1; echo "exit=$?" >> gpurun_out/r02j_fuzz.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1
