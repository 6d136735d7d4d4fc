#!/bin/bash
# Stage 2, A halves loaded by 1-CTA TMA onto each CTA's own barrier (no cross-CTA
# relay before the conversion); plus a dry run (synchronisation only, wrong dZ)
# to separate the sync latency from the rescale work.
mkdir -p gpurun_out/r2v
O=gpurun_out/r2v
timeout 300 python -m pytest tests/test_gpu_dz_q.py -k backward_row_skip -x -q -m gpu > $O/tests_skip.log 2>&1
rc=$?; echo "skip_test_rc=$rc"; tail -n 2 $O/tests_skip.log
[ $rc -ne 0 ] && exit 1
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for cfg in qwen7b; do
  for v in skip fused2 dry fused1; do
    case $v in skip*) E="RLHEAD_DZ_FUSED=0" ;; fused2*) E="RLHEAD_DZ_FUSED=2" ;; dry) E="RLHEAD_DZ_FUSED=2 RLHEAD_CVT_DRY=1" ;; fused1) E="RLHEAD_DZ_FUSED=1" ;; esac
    env $E timeout 900 python bench.py $AB --config $cfg > $O/ab_${cfg}_$v.json 2> $O/ab_${cfg}_$v.err
    echo "ab_${cfg}_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_${cfg}_$v.json')); k=d['kernels']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dh']['ms_total'], k['gemm_dw']['ms_total'], k.get('dz_from_q',{}).get('ms_total'))" 2>/dev/null)"
  done
done
