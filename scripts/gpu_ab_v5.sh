# v5 kernels: fused dH+dW launch and micro-batch size, same-box A/B.
mkdir -p gpurun_out
run() { label=$1; mb=$2; shift; shift
  env "$@" timeout -s KILL 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux --mb-rows $mb > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', d['value'], d['clocks']['sm_mhz'], {k:v['ms_total'] for k,v in d['kernels'].items() if 'gemm' in k})" 2>/dev/null || tail -c 800 gpurun_out/ab.log
}
run base16k 16384 X=1
run fused16k 16384 RLHEAD_FUSED_BWD=1
run base32k 32768 X=1
run base8k 8192 X=1
run base16k 16384 X=1
run fused16k 16384 RLHEAD_FUSED_BWD=1
run base32k 32768 X=1
run base8k 8192 X=1
