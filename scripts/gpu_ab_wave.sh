run() { # label env mb
  env $2 timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux --mb-rows $3 > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run red-16k RLHEAD_DW_RED=1 16384
run red-18944 RLHEAD_DW_RED=1 18944
run red-16k-fused "RLHEAD_DW_RED=1 RLHEAD_FUSED_BWD=1" 16384
run red-18944-fused "RLHEAD_DW_RED=1 RLHEAD_FUSED_BWD=1" 18944
run plain-64k RLHEAD_DW_RED=0 65536
run red-37888 RLHEAD_DW_RED=1 37888
run red-18944 RLHEAD_DW_RED=1 18944
