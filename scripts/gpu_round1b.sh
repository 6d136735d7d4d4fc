timeout -s KILL 1200 python bench.py > gpurun_out/bench_r1b.log 2>&1; echo "bench rc=$?"
timeout -s KILL 200 python scripts/probe.py --reps 1 > /dev/null 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 4 -c 4 -o gpurun_out/prof_gemm_r1b python scripts/probe.py --reps 1 > gpurun_out/ncu_full_r1b.log 2>&1; echo "ncu full rc=$?"
timeout -s KILL 300 python bench.py --max-mb 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/small4_r1b.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --max-mb 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_r1b.log 2>&1; echo "ncu launches rc=$?"
