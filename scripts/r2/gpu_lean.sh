#!/bin/bash
# Lean q epilogue + bounded dz grid: tests touching them, then same-box A/B
# q vs recompute (ratio vs r2d's 1.2586 isolates the q-path changes) and
# serial vs pipeline, then the HBM probe.
mkdir -p gpurun_out/r2h
O=gpurun_out/r2h
timeout 1500 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py tests/test_gpu_edge_branches.py tests/test_gpu_loss_variants.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in q recompute pipe q2; do
  case $v in
    q|q2) E=""; P=0 ;;
    recompute) E="RLHEAD_DZ_RECOMPUTE=1"; P=0 ;;
    pipe) E=""; P=1 ;;
  esac
  env $E timeout 900 python bench.py $AB --pipeline $P > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
timeout 600 python scripts/probe.py --config qwen7b --rows 16384 --reps 3 > $O/probe.json 2>&1
cat $O/probe.json
