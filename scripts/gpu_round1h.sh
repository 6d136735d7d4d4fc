# Final round-1 measurement at the v5 defaults (32k-row micro-batches) + the
# rewritten H1 kernels: bookkeeping parity, H1 probe (+ ncu per kernel), smoke,
# headline bench, ncu launch list of the same command, ncu --set full of the
# GEMMs, full GPU test suite.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "bookkeeping or tiny or empty or seq" > gpurun_out/h1_tests.log 2>&1; echo "h1 tests rc=$?"; tail -2 gpurun_out/h1_tests.log
timeout -s KILL 300 python scripts/probe_h1.py --reps 5 > gpurun_out/probe_h1.json 2>&1; echo "probe_h1 rc=$?"; tail -1 gpurun_out/probe_h1.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --print-units base --csv -k regex:"k_validate|k_flags|k_scan|k_compact" -s 4 -c 4 --log-file gpurun_out/ncu_h1.csv python scripts/probe_h1.py --reps 1 > /dev/null 2>&1; echo "ncu h1 rc=$?"
python scripts/ncu_metrics_table.py gpurun_out/ncu_h1.csv 2>/dev/null | tail -5
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v6.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_v6.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_v6.json 2> gpurun_out/bench_v6.err
echo "bench rc=$?"; tail -c 400 gpurun_out/bench_v6.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_v6.csv python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ncu_launches_v6.log 2>&1
echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 4 -c 4 -o gpurun_out/prof_gemm_v6 python scripts/probe.py --rows 32768 --reps 1 > gpurun_out/prof_gemm_v6.log 2>&1
echo "ncu full rc=$?"
timeout -s KILL 2400 python -m pytest tests -q -x -m gpu > gpurun_out/gpu_tests_v6.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_v6.log
