# Just-in-time tile claims (RLHEAD_SCHED_JIT=1): tests, ncu DRAM bytes, same-box A/B.
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest -q -x -m gpu tests/test_gpu_variants.py -k "bit_identical or sched-jit" > gpurun_out/jit_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/jit_tests.log
CMD="python scripts/probe.py --rows 16384 --reps 1"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for v in 0 1; do
  RLHEAD_SCHED_JIT=$v timeout -s KILL 400 ncu --metrics $M --clock-control none --print-units base -k regex:k_tc_gemm -s 4 -c 4 --csv --log-file gpurun_out/jit_$v.csv $CMD > /dev/null 2>&1
  echo "== jit=$v"; python scripts/ncu_metrics_table.py gpurun_out/jit_$v.csv 2>/dev/null | tail -4
done
run() { label=$1; shift
  env "$@" timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run base X=1
run jit RLHEAD_SCHED_JIT=1
run base X=1
run jit RLHEAD_SCHED_JIT=1
