# v5 defaults (dynamic scheduler, TMA dW reduce, TMA dZ stores, serpentine dW K):
# headline bench, ncu launch list, ncu --set full of the four GEMMs, full GPU tests.
mkdir -p gpurun_out
timeout -s KILL 1200 python bench.py > gpurun_out/bench_v5.json 2> gpurun_out/bench_v5.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_v5.json
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_v5.csv python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux > gpurun_out/ncu_launches_v5.log 2>&1
echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 4 -c 4 -o gpurun_out/prof_gemm_v5 python scripts/probe.py --rows 16384 --reps 1 > gpurun_out/prof_gemm_v5.log 2>&1
echo "ncu full rc=$?"
timeout -s KILL 2400 python -m pytest tests -q -x -m gpu > gpurun_out/gpu_tests_v5.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_v5.log
