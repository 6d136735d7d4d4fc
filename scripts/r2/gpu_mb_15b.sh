#!/bin/bash
# Micro-batch budget for the Qwen-1.5B head (h = 1536: per-micro-batch costs weigh more
# than at 7B): 16k (default) vs 32k vs 24k rows, same box.
mkdir -p gpurun_out/r2dd
O=gpurun_out/r2dd
AB="--config qwen1.5b --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in 16384 32768 24576 16384 32768 65536; do
  tag=mb$v; [ -f $O/ab_$tag.json ] && tag=${tag}_b
  timeout 900 python bench.py $AB --mb-rows $v > $O/ab_$tag.json 2> $O/ab_$tag.err
  echo "ab_$tag rc=$? $(python -c "import json; d=json.load(open('$O/ab_$tag.json')); k=d['kernels']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_lse']['ms_total'], k['gemm_dh']['ms_total'], k['gemm_dw']['ms_total'], k['dz_from_q']['ms_total'])" 2>/dev/null)"
done
