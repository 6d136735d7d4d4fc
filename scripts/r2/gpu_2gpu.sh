#!/bin/bash
# 2-GPU box: multi-GPU tests (vocab-parallel, DP dW modes, DP step vs the
# oracle), the bench's own --gpus 2 relaunch (Qwen-7B, OpenVLA) with per-
# phase times, the 1-GPU lines on the same box, and the pipeline A/B on GPU 0.
mkdir -p gpurun_out/r2_2gpu
O=gpurun_out/r2_2gpu
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_tp_symm.py tests/test_gpu_pipeline.py -q -m gpu --durations=10 > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests_2gpu.log
for cfg in qwen7b openvla; do
  for n in 1 2; do
    steps=10; [ $cfg = qwen7b ] && steps=3
    timeout 1500 python bench.py --gpus $n --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-aux --phases > $O/bench_${cfg}_dp$n.json 2> $O/bench_${cfg}_dp$n.err
    echo "$cfg dp$n rc=$? $(python -c "import json; d=json.load(open('$O/bench_${cfg}_dp$n.json')); print(d['n_gpus'], d['gpus_active'], d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['phases_ms'])" 2>/dev/null)"
  done
done
AB="--steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-aux"
for v in serial pipe; do
  case $v in serial*) P=0 ;; pipe*) P=1 ;; esac
  CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py $AB --pipeline $P > $O/ab_$v.json 2> $O/ab_$v.err
  echo "ab_$v rc=$? $(python -c "import json,sys; d=json.load(open('$O/ab_$v.json')); print(d['value'], d['clocks']['sm_mhz'])" 2>/dev/null)"
done
