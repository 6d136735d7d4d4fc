for c in qwen1.5b openvla; do
  timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c}_v3.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_${c}_v3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['roofline']['step_executed_frac_burst'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks']['sm_mhz'], d['aux']['fwd_only']['value'])"
done
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v3.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_v3.log | cut -c1-400
