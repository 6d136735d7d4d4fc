CMD="python scripts/probe.py --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout -s KILL 200 $CMD > /dev/null || exit 1
run() { label=$1; shift
  env "$@" timeout -s KILL 400 ncu --metrics $M --clock-control none -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/bwd_$label.csv $CMD > /dev/null 2>&1; echo "$label rc=$?"
}
run wide_g1_p1 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M_BWD=1
run wide_g1_p0 RLHEAD_L2_POLICY=0 RLHEAD_GROUP_M_BWD=1
run wide_g1_p2 RLHEAD_L2_POLICY=2 RLHEAD_GROUP_M_BWD=1
run wide_g2_p1 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M_BWD=2
run wide_g4_p0 RLHEAD_L2_POLICY=0 RLHEAD_GROUP_M_BWD=4
run narrow_g1_p1 RLHEAD_WIDE=0 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M_BWD=1
