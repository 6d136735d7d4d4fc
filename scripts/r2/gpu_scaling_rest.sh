#!/bin/bash
# Scaling of the remaining heads with the default NVLS dW sum: Qwen-1.5B head 1/2/4,
# OpenVLA head 2 (its 1 and 4 are in r2_end4).
mkdir -p gpurun_out/r2cc
O=gpurun_out/r2cc
for v in "qwen1.5b 1" "qwen1.5b 2" "qwen1.5b 4" "openvla 2" "qwen1.5b 4"; do
  set -- $v
  E="--steps 5 --warmup 3"
  [ $1 = openvla ] && E="--steps 20 --warmup 5 --mb-rows 32768 --split-groups 1"
  tag=$1_dp$2; [ -f $O/bench_$tag.json ] && tag=${tag}_b
  timeout 1200 python bench.py --config $1 --gpus $2 $E --no-cpu-baseline --no-aux --phases > $O/bench_$tag.json 2> $O/bench_$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/bench_$tag.json') if l.startswith('{')][-1]); print(d['n_gpus'], d['value'], (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'], d['config']['lpt_load_max_over_mean'], d['phases_ms']['micro_batches'], d['phases_ms']['dw_reduce'])" 2>/dev/null)"
done
