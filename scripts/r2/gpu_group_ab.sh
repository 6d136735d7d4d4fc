#!/bin/bash
# Forward raster group A/B in q + skip mode (16 pair-row tiles default).
mkdir -p gpurun_out/r2m
O=gpurun_out/r2m
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in g16 g25 g20 g16b; do
  case $v in g16|g16b) E="" ;; g25) E="RLHEAD_GROUP_M=50" ;; g20) E="RLHEAD_GROUP_M=40" ;; esac
  env $E timeout 900 python bench.py $AB > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'], {k: round(v['ms_total']/2) for k, v in d['kernels'].items() if k.startswith('gemm') or k == 'dz_from_q'})" 2>/dev/null)"
done
