CMD="python bench.py --max-mb 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CG2', d['value'], d['roofline']['step_executed_tflops'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 2 -c 2 -o gpurun_out/prof_cg2 $CMD > gpurun_out/ncu_cg2.log 2>&1; echo ncu rc=$?
