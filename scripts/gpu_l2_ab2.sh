CMD="python scripts/probe.py --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout -s KILL 120 python scripts/probe.py --reps 2
run() { label=$1; shift
  env "$@" timeout -s KILL 120 $CMD > gpurun_out/probe_$label.json 2>&1 && \
  env "$@" timeout -s KILL 600 ncu --metrics $M --clock-control none -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/l2_$label.csv $CMD > /dev/null 2>&1
  echo "== $label rc=$? $(cat gpurun_out/probe_$label.json | tail -1)"
}
run cg1_p1_g16 RLHEAD_CTA_GROUP=1 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=16
run cg2_p1_g16 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=16
run cg2_p0_g16 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=0 RLHEAD_GROUP_M=16
run cg2_p1_g32 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=32
run cg2_p1_g48 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=48
