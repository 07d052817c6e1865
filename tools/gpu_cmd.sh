for c in C2 C3 C5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/pipe_$c.json 2>>gpurun_out/pipe.err
done
