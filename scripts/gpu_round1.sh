set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout -s KILL 900 python bench.py > gpurun_out/bench_r1.log 2>&1; echo "bench rc=$?"
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r1.log 2>&1; echo "ref rc=$?"
timeout -s KILL 300 python bench.py --max-mb 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/small_r1.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 2 -c 4 -o gpurun_out/prof_gemm_r1 python bench.py --max-mb 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_r1.log 2>&1; echo "ncu full rc=$?"
timeout -s KILL 300 python bench.py --max-mb 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/small4_r1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --max-mb 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_r1.log 2>&1; echo "ncu launches rc=$?"
