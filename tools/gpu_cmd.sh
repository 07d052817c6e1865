for h in 0 1 2 3 0; do
  for c in C2 C3; do
    BITSORT_HINTS=$h timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/h${h}_$c.json 2>>gpurun_out/h.err
  done
done
