# Final check of the committed tree: full GPU suite, smoke, default bench.
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -x -m gpu > gpurun_out/gpu_tests_final.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_final.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
timeout -s KILL 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['step_executed_frac_burst'], d['cpu_baseline']['value'], d['gpu_launches'])" || tail -c 1500 gpurun_out/bench_final.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_reference.json
