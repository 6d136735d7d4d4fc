#!/bin/bash
# Final 1-GPU set on the round-2 tree: GPU suite, smoke, the default bench
# line (all legs), the ncu launch list of the same command (4 micro-batches),
# one ncu --set full capture per GEMM kind + dZ pass (16k micro-batch), HBM
# kernels (probe + ncu), cuBLAS same-shape comparison.
mkdir -p gpurun_out/r2i
O=gpurun_out/r2i
timeout 2400 python -m pytest tests -q -m gpu --durations=20 > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"; tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1
echo "smoke_rc=$?"; tail -n 3 $O/smoke.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench_rc=$?"
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2i/bench.json") if l.startswith("{")][-1])
print(d["value"], d["e2e"]["value"], d["clocks"], d["roofline"])
print(d["cpu_baseline"])
print(d["aux"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches.csv python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > $O/ncu_launches.log 2>&1
echo "ncu_launch_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_gemm|k_dz_from_q" -c 4 -o $O/prof_gemm python scripts/probe.py --config qwen7b --rows 16384 --reps 1 > $O/ncu_gemm.log 2>&1
echo "ncu_gemm_rc=$?"
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_flags_compact|k_validate|k_grpo_seg|k_merge|k_gather|k_dz_from_q" -c 14 -o $O/prof_hbm python scripts/probe_hbm.py --reps 1 > $O/ncu_hbm.log 2>&1
echo "ncu_hbm_rc=$?"
timeout 900 python scripts/probe.py --config qwen7b --rows 16384 --reps 3 --cublas --sustain 20 > $O/cublas_compare.json 2>&1
echo "cublas_rc=$?"; cat $O/cublas_compare.json
