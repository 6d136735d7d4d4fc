#!/bin/bash
# Backward-row skip (rows with dL/dlogp = 0 leave the dH/dW GEMMs): tests,
# then same-box A/B skip vs dense, for the Qwen-7B and Qwen-1.5B heads.
mkdir -p gpurun_out/r2j
O=gpurun_out/r2j
timeout 1800 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py tests/test_gpu_edge_branches.py tests/test_gpu_loss_variants.py tests/test_gpu_variants.py tests/test_gpu_streaming.py tests/test_gpu_dw_reduce_scatter.py tests/test_gpu_graph.py tests/test_gpu_hbm_kernels.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for cfg in qwen7b qwen1.5b; do
  for v in skip dense skip2; do
    case $v in skip*) E="RLHEAD_BWD_SKIP=1" ;; dense) E="RLHEAD_BWD_SKIP=0" ;; esac
    env $E timeout 900 python bench.py $AB --config $cfg > $O/ab_${cfg}_$v.json 2> $O/ab_${cfg}_$v.err
    echo "ab_${cfg}_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_${cfg}_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
  done
done
