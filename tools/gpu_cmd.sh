timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiset.py -x -q > gpurun_out/pytest_bal.log 2>&1; echo "exit=$?" >> gpurun_out/pytest_bal.log
for c in C5 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bal_$c.json 2>>gpurun_out/bal.err
done
