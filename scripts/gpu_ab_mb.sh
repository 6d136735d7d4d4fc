for mb in 65536 131072 65536 131072; do
  timeout -s KILL 900 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --mb-rows $mb 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb=$mb', d['value'], d['roofline']['step_executed_tflops'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k or k=='merge'})"
done
