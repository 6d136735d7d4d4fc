#!/bin/bash
# 1-GPU round-2 measurement set: dZ-from-q tests, the default bench line (all
# legs), the ncu launch list of the same command (short), one ncu --set full
# capture per kernel kind of a 16k micro-batch, the HBM probe, cuBLAS same-
# shape comparison, compute-sanitizer on the smoke + emulated reduce-scatter.
mkdir -p gpurun_out/r2e
O=gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_variants.py -q -m gpu -k "dz or fused_backward" > $O/dzq_tests.log 2>&1
echo "dzq_rc=$?"; tail -n 2 $O/dzq_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench_rc=$?"
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e']['value'], d['clocks'], d['roofline'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_launches.csv python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > $O/ncu_launches.log 2>&1
echo "ncu_launch_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_gemm|k_dz_from_q" -c 4 -o $O/prof_gemm python scripts/probe.py --config qwen7b --rows 16384 --reps 1 > $O/ncu_gemm.log 2>&1
echo "ncu_gemm_rc=$?"
timeout 600 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_flags_compact|k_validate|k_grpo_seg|k_merge|k_gather|k_dz_from_q" -c 14 -o $O/prof_hbm python scripts/probe_hbm.py --reps 1 > $O/ncu_hbm.log 2>&1
echo "ncu_hbm_rc=$?"
timeout 900 python scripts/probe.py --config qwen7b --rows 16384 --reps 3 --cublas --sustain 20 > $O/cublas_compare.json 2>&1
echo "cublas_rc=$?"; cat $O/cublas_compare.json
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 99 python -c "import __graft_entry__ as g; g.smoke()" > $O/san_smoke_$tool.log 2>&1
  echo "san smoke $tool rc=$?"
  timeout 1200 $CS --tool $tool --error-exitcode 99 python -m pytest -q -x tests/test_gpu_dw_reduce_scatter.py > $O/san_dwrs_$tool.log 2>&1
  echo "san dw_reduce_scatter $tool rc=$?"
done
