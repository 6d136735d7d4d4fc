#!/bin/bash
# Final 1-GPU check of the round-2 tree: whole GPU suite, smoke, default bench line
# (all legs), the other heads' default lines.
mkdir -p gpurun_out/r2y
O=gpurun_out/r2y
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"; tail -n 3 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "smoke_rc=$?"; tail -n 1 $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench_rc=$? $(python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'])" 2>/dev/null)"
for cfg in qwen1.5b openvla; do
  timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-aux > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('$O/bench_$cfg.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'])" 2>/dev/null)"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo "ref rc=$? $(tail -c 300 $O/bench_reference.json)"
