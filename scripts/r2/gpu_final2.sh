#!/bin/bash
# Final 1-GPU check of the round-2 tree (skip mode default): GPU suite, smoke,
# the default bench line with all legs, the ncu launch list of the same
# command, full ncu captures of the GEMMs + dZ pass in skip mode, other heads.
mkdir -p gpurun_out/r2n
O=gpurun_out/r2n
timeout 2400 python -m pytest tests -q -m gpu --durations=20 > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"; tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke_rc=$?"; tail -n 3 $O/smoke.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench_rc=$?"
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2n/bench.json") if l.startswith("{")][-1])
print(d["value"], d["e2e"]["value"], d["clocks"], d["roofline"])
print(d["cpu_baseline"]["value"], d["aux"]["torch_eager_reference"]["value"], d["aux"]["fwd_only"]["value"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches.csv python bench.py --max-mb 6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > $O/ncu_launches.log 2>&1
echo "ncu_launch_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_gemm|k_dz_from_q|k_keep_compact" -c 5 -o $O/prof_gemm python scripts/probe.py --config qwen7b --rows 32768 --reps 1 > $O/ncu_gemm.log 2>&1
echo "ncu_gemm_rc=$?"
for cfg in qwen1.5b openvla; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/bench_$cfg.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])" 2>/dev/null)"
done
