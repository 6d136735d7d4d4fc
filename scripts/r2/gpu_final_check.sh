#!/bin/bash
# Last check of the committed tree on one GPU: whole GPU suite + smoke + a short default bench.
mkdir -p gpurun_out/r2_last
O=gpurun_out/r2_last
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_suite.log 2>&1
echo "suite_rc=$?"; tail -n 2 $O/gpu_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "smoke_rc=$?"; tail -n 1 $O/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-aux > $O/bench.json 2> $O/bench.err
echo "bench_rc=$? $(python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'])" 2>/dev/null)"
