#!/bin/bash
# OpenVLA strong scaling at 4 GPUs (114,688 tokens per step, ~17 ms steps):
# micro-batch budget (16k vs 32k rows: one micro-batch per rank) and sharding
# (whole groups vs single sequences with all-reduced group statistics).
mkdir -p gpurun_out/r2_vla
O=gpurun_out/r2_vla
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases"
for v in "1 16384 0" "1 32768 0" "4 16384 0" "4 32768 0" "4 32768 1" "4 16384 1" "2 32768 1" "2 32768 0"; do
  set -- $v
  n=$1; mb=$2; sp=$3
  tag=n${n}_mb${mb}_split${sp}
  timeout 900 python bench.py --gpus $n $B --mb-rows $mb --split-groups $sp > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['config']['lpt_load_max_over_mean'], d['phases_ms']['micro_batches'], d['phases_ms']['dw_reduce'])" 2>/dev/null)"
done
