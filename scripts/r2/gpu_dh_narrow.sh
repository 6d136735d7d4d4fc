#!/bin/bash
# dH on 256-wide tiles (798 tiles = 10.8 waves of 74 pairs per 16k micro-batch instead of
# 399 = 5.4 waves of 512-wide) vs the default, same box; plus the dH test variant.
mkdir -p gpurun_out/r2bb
O=gpurun_out/r2bb
RLHEAD_WIDE_DH=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > $O/tests_narrow_dh.log 2>&1
rc=$?; echo "tests_rc=$rc"; tail -n 2 $O/tests_narrow_dh.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in wide narrow wide2 narrow2; do
  case $v in wide*) E="RLHEAD_WIDE_DH=1" ;; narrow*) E="RLHEAD_WIDE_DH=0" ;; esac
  env $E timeout 900 python bench.py $AB > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json; d=json.load(open('$O/ab_$v.json')); k=d['kernels']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_lse']['ms_total'], k['gemm_dh']['ms_total'], k['gemm_dw']['ms_total'])" 2>/dev/null)"
done
