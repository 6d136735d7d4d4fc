#!/bin/bash
# OpenVLA 4-GPU fixed costs: fused reduce-scatter (symm) vs NCCL, full vs shard dW
# output, per-phase max AND min over ranks; 2-GPU DP tests.
mkdir -p gpurun_out/r2w
O=gpurun_out/r2w
timeout 900 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests_2gpu.log
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases --mb-rows 32768 --split-groups 1"
for v in "1 symm full" "4 symm shard" "4 nccl shard" "4 nccl full" "4 symm full" "4 symm shard"; do
  set -- $v
  n=$1; coll=$2; out=$3
  tag=n${n}_${coll}_${out}
  [ -f $O/$tag.json ] && tag=${tag}_b
  timeout 900 python bench.py --gpus $n $B --collective $coll --dw-output $out > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); k=d['kernels']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dw']['ms_total'], k['gemm_lse']['ms_total'], k['gemm_dh']['ms_total'], d['phases_ms'])" 2>/dev/null)"
done
