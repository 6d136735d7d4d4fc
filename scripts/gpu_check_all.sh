# full GPU suite + a short bench (merge/aux numbers)
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout -s KILL 600 python bench.py --config qwen1.5b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_check.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_check.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], json.dumps(d['aux']))"
