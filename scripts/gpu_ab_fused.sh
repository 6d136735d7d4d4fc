for v in "RLHEAD_FUSED_BWD=1" "RLHEAD_FUSED_BWD=0" "RLHEAD_FUSED_BWD=1" "RLHEAD_FUSED_BWD=0"; do
  env $v timeout -s KILL 900 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['step_executed_tflops'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k or k=='merge'})"
done
