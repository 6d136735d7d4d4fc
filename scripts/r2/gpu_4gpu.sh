#!/bin/bash
# 4-GPU scaling on one box: Qwen-7B head and OpenVLA head at N = 1, 2, 4
# (bench's own relaunch), per-phase times; the 2-rank DP-vs-oracle test.
mkdir -p gpurun_out/${OUT:-r2_4gpu}
O=gpurun_out/${OUT:-r2_4gpu}
nvidia-smi topo -m > $O/topo.txt 2>&1
for cfg in openvla qwen7b; do
  for n in 1 2 4; do
    steps=10; [ $cfg = qwen7b ] && steps=3
    timeout 1500 python bench.py --gpus $n --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-aux --phases > $O/bench_${cfg}_dp$n.json 2> $O/bench_${cfg}_dp$n.err
    echo "$cfg dp$n rc=$? $(python -c "import json; d=json.load(open('$O/bench_${cfg}_dp$n.json')); print(d['n_gpus'], d['gpus_active'], d['value'], d['clocks']['sm_mhz'], d['phases_ms'])" 2>/dev/null)"
  done
done
