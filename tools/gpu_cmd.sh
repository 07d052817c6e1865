for c in C3 C5 C4 C2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tmpl_$c.json 2>>gpurun_out/tmpl.err
done
