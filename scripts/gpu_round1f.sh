timeout -s KILL 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout -s KILL 1200 python bench.py > gpurun_out/bench_r1f.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r1f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']), d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'], d['step_ms_rank0'], d['gpu_launches'], json.dumps(d['aux']))"
timeout -s KILL 300 python scripts/probe.py --rows 16384 --reps 1 > gpurun_out/probe16k.json 2>&1; echo "probe rc=$?"; tail -1 gpurun_out/probe16k.json
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 4 -c 4 -o gpurun_out/prof_gemm_v4 python scripts/probe.py --rows 16384 --reps 1 > gpurun_out/ncu_gemm_v4.log 2>&1; echo "ncu rc=$?"
