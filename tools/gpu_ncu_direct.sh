M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,lts__t_sector_op_red_hit_rate.pct,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum
for c in C2 C4; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:"scatter|scan" -c 4 --csv --log-file gpurun_out/ncu_direct_$c.csv \
      python tools/run_one.py --config $c --path DIRECT --iters 2 > gpurun_out/ncu_direct_$c.log 2>&1
done
