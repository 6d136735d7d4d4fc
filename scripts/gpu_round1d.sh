timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout -s KILL 1200 python bench.py > gpurun_out/bench_r1d.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r1d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'], d['step_ms_rank0'], json.dumps(d['aux']))"
CMD="python bench.py --max-mb 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_merge -s 4 -c 1 -o gpurun_out/prof_merge_r1d $CMD > gpurun_out/ncu_merge.log 2>&1; echo "ncu merge rc=$?"
