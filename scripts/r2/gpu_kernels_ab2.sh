#!/bin/bash
# Round-2 kernels v2 (H1 walk + 1024/4096-row tiles, persistent float4 merge,
# shuffle-scan segmented GRPO): GPU suite, smoke, HBM probe + ncu, and the
# forward raster-group A/B (smaller groups) + fused backward, same box.
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"
tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke_rc=$?"
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2> $O/probe_hbm.err
echo "probe_rc=$?"; cat $O/probe_hbm.json
timeout 900 ncu --set full --clock-control none -k regex:"k_flags_compact|k_validate|k_grpo_seg|k_merge|k_gather" -c 12 -o $O/prof_hbm python scripts/probe_hbm.py --reps 1 > $O/ncu_hbm.log 2>&1
echo "ncu_rc=$?"
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in base g8 g12 fused base2; do
  case $v in
    base|base2) E="" ;;
    fused) E="RLHEAD_FUSED_BWD=1" ;;
    g8) E="RLHEAD_GROUP_M=16" ;;
    g12) E="RLHEAD_GROUP_M=24" ;;
  esac
  env $E timeout 900 python bench.py $AB > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
