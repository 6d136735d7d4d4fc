CMD="python bench.py --max-mb 1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
run() { # $1 = label, rest = env
  label=$1; shift
  env "$@" timeout -s KILL 200 $CMD > /dev/null 2>&1 && \
  env "$@" timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:k_tc_gemm -s 1 -c 4 --csv $CMD 2>/dev/null | grep k_tc_gemm > gpurun_out/l2_$label.csv
  echo "== $label rc=$?"
}
run cg1_p1_g16 RLHEAD_CTA_GROUP=1 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=16
run cg2_p1_g16 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=16
run cg2_p0_g16 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=0 RLHEAD_GROUP_M=16
run cg2_p1_g32 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=1 RLHEAD_GROUP_M=32
run cg2_p0_g8 RLHEAD_CTA_GROUP=2 RLHEAD_L2_POLICY=0 RLHEAD_GROUP_M=8
for cg in 1 2; do
  RLHEAD_CTA_GROUP=$cg timeout -s KILL 300 python bench.py --max-mb 16 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CG$cg', d['value'], d['roofline']['step_executed_tflops'], d['clocks'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})"
done
