#!/bin/bash
# Fused-backward stage 2 (RLHEAD_DZ_FUSED=2: q rescaled into dZ by converter warps inside
# the dH / dW GEMMs, no k_dz_from_q pass): bit-identity tests first (short timeout: a
# barrier bug would hang), then same-box A/B against the default skip mode and stage 1.
mkdir -p gpurun_out/r2s
O=gpurun_out/r2s
timeout 300 python -m pytest tests/test_gpu_dz_q.py -k backward_row_skip -x -q -m gpu > $O/tests_skip.log 2>&1
rc=$?; echo "skip_test_rc=$rc"; tail -n 5 $O/tests_skip.log
[ $rc -ne 0 ] && exit 1
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_dz_q.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 5 $O/tests.log
RLHEAD_DZ_FUSED=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edge_branches.py tests/test_gpu_pipeline.py -q -m gpu > $O/tests_env2.log 2>&1
echo "tests_env2_rc=$?"; tail -n 5 $O/tests_env2.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for cfg in qwen7b qwen1.5b; do
  for v in skip fused2 fused1 skip2 fused2b; do
    case $v in skip*) E="RLHEAD_DZ_FUSED=0" ;; fused1) E="RLHEAD_DZ_FUSED=1" ;; fused2*) E="RLHEAD_DZ_FUSED=2" ;; esac
    env $E timeout 900 python bench.py $AB --config $cfg > $O/ab_${cfg}_$v.json 2> $O/ab_${cfg}_$v.err
    echo "ab_${cfg}_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_${cfg}_$v.json')); k=d['kernels']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dh']['ms_total'], k['gemm_dw']['ms_total'], k.get('dz_from_q',{}).get('ms_total'))" 2>/dev/null)"
  done
done
