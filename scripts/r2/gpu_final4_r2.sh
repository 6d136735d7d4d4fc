#!/bin/bash
# End-of-round multi-GPU check (default collective nvls): multi-GPU tests on 2 of the
# 4 GPUs, Qwen-7B head at 1/2/4 GPUs, Qwen-32B head at 4, OpenVLA head at 1/4.
mkdir -p gpurun_out/r2_end4
O=gpurun_out/r2_end4
CUDA_VISIBLE_DEVICES=0,1 timeout 1800 python -m pytest tests/test_gpu_tp_symm.py tests/test_gpu_streaming.py tests/test_gpu_dw_reduce_scatter.py -q -m gpu > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 2 $O/tests_2gpu.log
for v in "qwen7b 1" "qwen7b 2" "qwen7b 4" "qwen32b 4" "openvla 1" "openvla 4"; do
  set -- $v
  E=""; [ $1 = qwen32b ] && E="--no-e2e"   # 54 GB of pinned host hidden per rank otherwise
  [ $1 = openvla ] && E="--steps 20 --warmup 5 --mb-rows 32768 --split-groups 1"
  timeout 1800 python bench.py --config $1 --gpus $2 --steps 3 --warmup 3 --no-cpu-baseline --no-aux --phases $E > $O/bench_$1_dp$2.json 2> $O/bench_$1_dp$2.err
  echo "$1 dp$2 rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/bench_$1_dp$2.json') if l.startswith('{')][-1]); print(d['n_gpus'], d['value'], (d['e2e'] or {}).get('value'), d['clocks']['sm_mhz'], d['config']['lpt_load_max_over_mean'], d['phases_ms']['micro_batches'], d['phases_ms']['dw_reduce'])" 2>/dev/null)"
done
