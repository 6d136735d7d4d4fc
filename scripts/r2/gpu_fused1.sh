#!/bin/bash
# Fused-backward stage 1 (RLHEAD_DZ_FUSED=1: rows partitioned A != 0 first, backward
# over that prefix in place): tests, then same-box A/B against the default skip mode.
mkdir -p gpurun_out/r2r
O=gpurun_out/r2r
timeout 1200 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 5 $O/tests.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for cfg in qwen7b qwen1.5b; do
  for v in skip fused skip2; do
    case $v in skip*) E="RLHEAD_DZ_FUSED=0" ;; fused) E="RLHEAD_DZ_FUSED=1" ;; esac
    env $E timeout 900 python bench.py $AB --config $cfg > $O/ab_${cfg}_$v.json 2> $O/ab_${cfg}_$v.err
    echo "ab_${cfg}_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_${cfg}_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['kernels']['dz_from_q']['ms_total'])" 2>/dev/null)"
  done
done
