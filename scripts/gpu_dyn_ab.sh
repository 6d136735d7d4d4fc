# Dynamic tile scheduler A/B: variant + bit-identity tests, ncu DRAM bytes per
# GEMM on one 16k-row micro-batch, then same-box bench runs.
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest -q -x tests/test_gpu_variants.py -k "dyn or bit_identical" > gpurun_out/variants_dyn.log 2>&1
echo "variants rc=$?"; tail -3 gpurun_out/variants_dyn.log
CMD="python scripts/probe.py --rows 16384 --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
prof() { label=$1; shift
  env "$@" timeout -s KILL 400 ncu --metrics $M --clock-control none --print-units base -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/dyn_$label.csv $CMD > /dev/null 2>&1
  echo "== $label rc=$?"
  python scripts/ncu_metrics_table.py gpurun_out/dyn_$label.csv 2>/dev/null | tail -4
}
prof base X=1
prof dyn RLHEAD_DYN_SCHED=1
prof dyn_tma RLHEAD_DYN_SCHED=1 RLHEAD_DW_RED=2
prof dyn_g8 RLHEAD_DYN_SCHED=1 RLHEAD_GROUP_M=16
run() { label=$1; shift
  env "$@" timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run base X=1
run dyn RLHEAD_DYN_SCHED=1
run dyn_tma RLHEAD_DYN_SCHED=1 RLHEAD_DW_RED=2
run base X=1
run dyn RLHEAD_DYN_SCHED=1
run dyn_tma RLHEAD_DYN_SCHED=1 RLHEAD_DW_RED=2
