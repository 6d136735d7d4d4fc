#!/bin/bash
# Round-2 kernels (H1 single-pass scan, segmented GRPO, merge batches of 8,
# fused dH+dW with TMA reduce + serpentine dW): GPU suite, smoke, same-box
# bench A/B (fused backward, forward raster group), HBM probe + ncu.
mkdir -p gpurun_out/r2b
O=gpurun_out/r2b
timeout 2400 python -m pytest tests -q -m gpu -x --durations=25 > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"
tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke_rc=$?"
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2> $O/probe_hbm.err
echo "probe_rc=$?"
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in base fused g48 base2 fused2; do
  case $v in
    base|base2) E="" ;;
    fused|fused2) E="RLHEAD_FUSED_BWD=1" ;;
    g48) E="RLHEAD_GROUP_M=96" ;;
  esac
  env $E timeout 900 python bench.py $AB > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
timeout 900 ncu --set full --clock-control none -k regex:"k_flags_compact|k_validate|k_grpo_seg|k_merge|k_gather" -c 12 -o $O/prof_hbm python scripts/probe_hbm.py --reps 1 > $O/ncu_hbm.log 2>&1
echo "ncu_rc=$?"
