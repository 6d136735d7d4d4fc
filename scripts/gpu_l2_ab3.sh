# Per-operand TMA L2 hints for the backward GEMMs (RLHEAD_L2_<KIND>="ab",
# 0 normal / 1 evict_last / 2 evict_first): ncu DRAM bytes per kernel on one
# 16k-row micro-batch, then same-box bench A/B.
mkdir -p gpurun_out
CMD="python scripts/probe.py --rows 16384 --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout -s KILL 200 $CMD > gpurun_out/probe_base.json 2>&1 || { echo probe failed; tail -20 gpurun_out/probe_base.json; exit 1; }
prof() { label=$1; shift
  env "$@" timeout -s KILL 400 ncu --metrics $M --clock-control none --print-units base -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/l2v_$label.csv $CMD > /dev/null 2>&1
  echo "== $label rc=$?"
  python scripts/ncu_metrics_table.py gpurun_out/l2v_$label.csv 2>/dev/null | tail -6
}
prof base
prof dw21 RLHEAD_L2_DW=21
prof dw01 RLHEAD_L2_DW=01
prof dw22 RLHEAD_L2_DW=22
prof dw12 RLHEAD_L2_DW=12
prof dh21 RLHEAD_L2_DH=21
prof dh12 RLHEAD_L2_DH=12
prof dh20 RLHEAD_L2_DH=20
prof dz00 RLHEAD_L2_DZ=00 RLHEAD_L2_FWD=00
run() { # label env...
  label=$1; shift
  env "$@" timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run base X=1
run dw21 RLHEAD_L2_DW=21
run dw21dh21 RLHEAD_L2_DW=21 RLHEAD_L2_DH=21
run base X=1
run dw21 RLHEAD_L2_DW=21
