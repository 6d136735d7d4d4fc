CMD="python scripts/probe.py --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout -s KILL 200 $CMD && timeout -s KILL 900 ncu --metrics $M --clock-control none -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/l2_wide.csv $CMD; echo rc=$?
