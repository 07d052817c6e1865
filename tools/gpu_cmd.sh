for c in C5 C4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/kpt_sel_$c.json 2>>gpurun_out/kpt20.err
done
