for v in dist a2a p2p push; do
  timeout 300 python bench.py --config C2 --$v --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/v_$v.json 2> gpurun_out/v_$v.err
  echo "$v exit=$?" >> gpurun_out/v_exit.log
done
