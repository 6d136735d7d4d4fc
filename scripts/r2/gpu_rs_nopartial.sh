#!/bin/bash
# Fused reduce-scatter with no_partial (a rank's only micro-batch does not read
# grad_weight) + bulk copies vs the NVLS sum; OpenVLA at 4 GPUs; tests.
mkdir -p gpurun_out/r2aa
O=gpurun_out/r2aa
timeout 600 python -m pytest tests/test_gpu_dw_reduce_scatter.py -q -m gpu > $O/tests_rs.log 2>&1
rc=$?; echo "rs_tests_rc=$rc"; tail -n 2 $O/tests_rs.log
[ $rc -ne 0 ] && exit 1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu > $O/tests_2gpu.log 2>&1
echo "tests_2gpu_rc=$?"; tail -n 2 $O/tests_2gpu.log
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases --mb-rows 32768 --split-groups 1"
for v in "1 nvls full" "4 symm shard" "4 nvls shard" "4 symm full" "4 nvls full" "4 symm shard" "4 nvls shard"; do
  set -- $v
  n=$1; coll=$2; out=$3
  tag=n${n}_${coll}_${out}
  [ -f $O/$tag.json ] && tag=${tag}_b
  timeout 900 python bench.py --gpus $n $B --collective $coll --dw-output $out > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); k=d['kernels']; p=d['phases_ms']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dw']['ms_total'], k['misc']['ms_total'], p['micro_batches'], p.get('min_over_ranks',{}).get('micro_batches'), p['dw_reduce'])" 2>/dev/null)"
done
