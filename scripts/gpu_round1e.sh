timeout -s KILL 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r1e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_r1e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], json.dumps(d['aux']))"
