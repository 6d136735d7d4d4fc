#!/bin/bash
# Micro-batch size A/B in skip mode (16k / 24k / 32k rows), GRPO kernel probe,
# same box.
mkdir -p gpurun_out/r2k
O=gpurun_out/r2k
timeout 600 python -m pytest tests/test_gpu_hbm_kernels.py tests/test_gpu_advantage.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 2 $O/tests.log
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2>&1
python -c "import json; d=json.load(open('$O/probe_hbm.json')); print(d['h2_grpo'], d['h1_whole_batch']['ms'])"
timeout 900 ncu --set full --clock-control none -k regex:"k_grpo_seg" -c 2 -o $O/prof_grpo python scripts/probe_hbm.py --reps 1 > $O/ncu_grpo.log 2>&1
echo "ncu_rc=$?"
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in 16384 24576 32768 16384b; do
  mb=${v%b}
  timeout 900 python bench.py $AB --mb-rows $mb > $O/ab_mb$v.json 2> $O/ab_mb$v.err
  echo "ab_mb$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_mb$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
