# v6 kernels on the other BASELINE configs (1 GPU): Qwen-1.5B head, OpenVLA head.
mkdir -p gpurun_out
for cfg in qwen1.5b openvla; do
  timeout -s KILL 1200 python bench.py --config $cfg > gpurun_out/bench_v6_$cfg.json 2> gpurun_out/bench_v6_$cfg.err; echo "$cfg rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_v6_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_executed_frac_burst'], d['cpu_baseline']['value'])" || tail -c 1500 gpurun_out/bench_v6_$cfg.err
done
# dH serpentine K A/B (Qwen-7B, 16k rows)
CMD="python scripts/probe.py --rows 16384 --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for v in 0 1; do
  RLHEAD_DH_SERP=$v timeout -s KILL 400 ncu --metrics $M --clock-control none --print-units base -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/dhserp_$v.csv $CMD > /dev/null 2>&1
  echo "== dh_serp=$v"; python scripts/ncu_metrics_table.py gpurun_out/dhserp_$v.csv 2>/dev/null | tail -4
done
run() { label=$1; shift
  env "$@" timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run base X=1
run dhserp RLHEAD_DH_SERP=1
run base X=1
run dhserp RLHEAD_DH_SERP=1
