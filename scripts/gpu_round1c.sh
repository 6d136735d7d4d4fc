# headline bench + launch list + ncu full capture of the merge kernel
timeout -s KILL 1200 python bench.py > gpurun_out/bench_r1c.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r1c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'], d['step_ms_rank0'])"
CMD="python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
timeout -s KILL 600 $CMD > gpurun_out/plain_mb4.log 2>&1; echo "plain rc=$?"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_merge -s 4 -c 1 -o gpurun_out/prof_merge_r1c $CMD > gpurun_out/ncu_merge.log 2>&1; echo "ncu merge rc=$?"
