#!/bin/bash
# The per-head bench defaults (micro-batch budget, OpenVLA sequence sharding) as the
# driver would run them: no tuning flags.
mkdir -p gpurun_out/r2ee
O=gpurun_out/r2ee
for v in "openvla 1" "openvla 4" "qwen1.5b 1" "qwen1.5b 4"; do
  set -- $v
  timeout 1200 python bench.py --config $1 --gpus $2 --no-cpu-baseline --no-aux > $O/bench_$1_dp$2.json 2> $O/bench_$1_dp$2.err
  echo "$1 dp$2 rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/bench_$1_dp$2.json') if l.startswith('{')][-1]); c=d['config']; print(d['n_gpus'], d['value'], (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'], c['micro_batch_rows'], c.get('sharding'), c['lpt_load_max_over_mean'])" 2>/dev/null)"
done
