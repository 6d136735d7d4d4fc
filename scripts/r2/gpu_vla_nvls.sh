#!/bin/bash
# DP dW sum after the last dW GEMM through the NVSwitch (collective nvls:
# multimem.ld_reduce of each owned slab) vs NCCL vs the fused epilogue reduce-scatter,
# full and sharded dW output; OpenVLA at 4 GPUs, Qwen-7B at 4 GPUs; 2-GPU DP tests.
mkdir -p gpurun_out/r2x
O=gpurun_out/r2x
timeout 900 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests_2gpu.log
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases --mb-rows 32768 --split-groups 1"
for v in "1 symm full" "4 nvls shard" "4 nccl shard" "4 nvls full" "4 nccl full" "4 nvls shard" "4 symm shard"; do
  set -- $v
  n=$1; coll=$2; out=$3
  tag=n${n}_${coll}_${out}
  [ -f $O/$tag.json ] && tag=${tag}_b
  timeout 900 python bench.py --gpus $n $B --collective $coll --dw-output $out > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); k=d['kernels']; p=d['phases_ms']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dw']['ms_total'], k['misc']['ms_total'], p['micro_batches'], p['dw_reduce'], p.get('min_over_ranks',{}).get('dw_reduce'))" 2>/dev/null)"
done
B7="--config qwen7b --steps 2 --warmup 3 --no-cpu-baseline --no-aux --phases"
for coll in nvls symm; do
  timeout 1200 python bench.py --gpus 4 $B7 --collective $coll > $O/qwen7b_n4_$coll.json 2> $O/qwen7b_n4_$coll.err
  echo "qwen7b_n4_$coll rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/qwen7b_n4_$coll.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['phases_ms']['dw_reduce'])" 2>/dev/null)"
done
