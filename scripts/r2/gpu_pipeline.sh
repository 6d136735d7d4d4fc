#!/bin/bash
# Split API + two-stream pipeline: tests, then same-box bench A/B (serial vs
# pipelined), then the default bench line with all legs, HBM probe.
mkdir -p gpurun_out/r2g
O=gpurun_out/r2g
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_dz_q.py tests/test_gpu_hbm_kernels.py tests/test_gpu_parity.py tests/test_gpu_advantage.py tests/test_gpu_streaming.py tests/test_gpu_graph.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests.log
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in serial pipe serial2 pipe2; do
  case $v in serial*) P=0 ;; pipe*) P=1 ;; esac
  timeout 900 python bench.py $AB --pipeline $P > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2>&1
echo "probe_rc=$?"
