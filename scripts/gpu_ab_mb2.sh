for mb in ${MBS:-65536 131072 65536 131072}; do
  timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux --mb-rows $mb > gpurun_out/ab_mb_$mb.log 2>&1; echo "mb=$mb rc=$?"
  tail -1 gpurun_out/ab_mb_$mb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mb=$mb', d['value'], d['roofline']['step_executed_tflops'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 1500 gpurun_out/ab_mb_$mb.log
done
