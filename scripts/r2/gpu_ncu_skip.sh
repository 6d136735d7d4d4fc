#!/bin/bash
# ncu evidence for the default (skip-mode) path on representative micro-
# batches (the layout's first ones are the forced A = 0 groups): launch list of
# the bench command on micro-batches 10..15, one --set full capture per kernel
# of micro-batch 10 (16k rows), cuBLAS same-shape comparison there.
mkdir -p gpurun_out/r2p
O=gpurun_out/r2p
timeout 900 python bench.py --max-mb 16 --mb-offset 40 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > $O/bench_short.json 2>&1
echo "bench_short_rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/ncu_launches.csv python bench.py --max-mb 16 --mb-offset 40 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > $O/ncu_launches.log 2>&1
echo "ncu_launch_rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_gemm|k_dz_from_q|k_keep_compact" -c 5 -o $O/prof_gemm python scripts/probe.py --config qwen7b --rows 16384 --mb-index 10 --reps 1 > $O/ncu_gemm.log 2>&1
echo "ncu_gemm_rc=$?"
timeout 900 python scripts/probe.py --config qwen7b --rows 16384 --mb-index 10 --reps 3 --cublas --sustain 20 > $O/cublas_compare.json 2>&1
echo "cublas_rc=$?"; cat $O/cublas_compare.json
