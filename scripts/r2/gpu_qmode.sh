#!/bin/bash
# q-mode backward (forward epilogue stores q = e^{z - m_tile}; k_dz_from_q
# replaces the dZ recompute GEMM): new tests first, then the whole GPU suite,
# smoke, and same-box bench A/B: q vs recompute, fused vs separate dH/dW.
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
timeout 1200 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_hbm_kernels.py tests/test_gpu_parity.py -q -m gpu -x > $O/new_tests.log 2>&1
echo "new_rc=$?"; tail -n 3 $O/new_tests.log
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"; tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke_rc=$?"
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in q recompute q_fused q2; do
  case $v in
    q|q2) E="" ;;
    recompute) E="RLHEAD_DZ_RECOMPUTE=1" ;;
    q_fused) E="RLHEAD_FUSED_BWD=1" ;;
  esac
  env $E timeout 900 python bench.py $AB > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
done
for it in 4 8 16; do
  RLHEAD_H1_ITEMS=$it timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm_items$it.json 2>&1
  echo "probe items=$it $(python -c "import json; d=json.load(open('$O/probe_hbm_items$it.json')); print(d['h1_whole_batch']['ms'], d['h2_grpo']['ms'], d['micro_batch'].get('merge'), d['micro_batch'].get('dz_from_q'))" 2>/dev/null)"
done
