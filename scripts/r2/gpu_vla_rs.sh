#!/bin/bash
# OpenVLA 4-GPU: the fused dW reduce-scatter epilogue on 256-wide double-buffered tiles
# (RLHEAD_RS_NARROW=1, default) vs 512-wide single-buffered, and the sharded-gradient
# output (--dw-output shard: no broadcast); 2-GPU DP tests incl. the shard mode.
mkdir -p gpurun_out/r2t
O=gpurun_out/r2t
timeout 900 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests_2gpu.log
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases --mb-rows 32768 --split-groups 1"
for v in "1 1 full" "4 0 full" "4 1 full" "4 1 shard" "4 0 full" "2 1 full" "2 1 shard"; do
  set -- $v
  n=$1; nar=$2; out=$3
  tag=n${n}_narrow${nar}_${out}
  [ -f $O/$tag.json ] && tag=${tag}_b
  RLHEAD_RS_NARROW=$nar timeout 900 python bench.py --gpus $n $B --dw-output $out > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); k=d['kernels']; print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['phases_ms']['micro_batches'], d['phases_ms']['dw_reduce'], k['gemm_dw']['ms_total'], k['misc']['ms_total'])" 2>/dev/null)"
done
B7="--config qwen7b --steps 2 --warmup 3 --no-cpu-baseline --no-aux --phases"
for n in 4; do
  timeout 1200 python bench.py --gpus $n $B7 > $O/qwen7b_n$n.json 2> $O/qwen7b_n$n.err
  echo "qwen7b_n$n rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/qwen7b_n$n.json') if l.startswith('{')][-1]); print(d['value'], d['clocks']['sm_mhz'], d['phases_ms'])" 2>/dev/null)"
done
