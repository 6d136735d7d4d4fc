#!/bin/bash
# Micro-batch size A/B (skip mode), smaller budgets, same box.
mkdir -p gpurun_out/r2l
O=gpurun_out/r2l
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in 16384 12288 8192 20480 16384b; do
  mb=${v%b}
  timeout 900 python bench.py $AB --mb-rows $mb > $O/ab_mb$v.json 2> $O/ab_mb$v.err
  echo "ab_mb$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_mb$v.json')); print(d['value'], d['clocks']['sm_mhz'], d['roofline']['kernel'], d['roofline']['frac'], {k: round(v['ms_total']/2) for k, v in d['kernels'].items() if k.startswith('gemm') or k == 'dz_from_q'})" 2>/dev/null)"
done
