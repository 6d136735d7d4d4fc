#!/bin/bash
# Fused epilogue reduce-scatter with whole-line bulk copies (RLHEAD_RS_BULK=1) vs
# 16-B stores vs the NVLS sum after the GEMM; OpenVLA at 4 GPUs; emulated and
# 2-GPU tests with the bulk path.
mkdir -p gpurun_out/r2z
O=gpurun_out/r2z
timeout 600 python -m pytest tests/test_gpu_dw_reduce_scatter.py -q -m gpu > $O/tests_rs.log 2>&1
rc=$?; echo "rs_tests_rc=$rc"; tail -n 2 $O/tests_rs.log
[ $rc -ne 0 ] && exit 1
RLHEAD_RS_BULK=1 timeout 900 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu -k "fused or streaming" > $O/tests_2gpu_bulk.log 2>&1
echo "tests_2gpu_bulk_rc=$?"; tail -n 2 $O/tests_2gpu_bulk.log
B="--config openvla --steps 20 --warmup 5 --no-cpu-baseline --no-aux --phases --mb-rows 32768 --split-groups 1"
for v in "1 nvls full 0" "4 symm shard 1" "4 nvls shard 0" "4 symm full 1" "4 nvls full 0" "4 symm shard 0" "4 symm shard 1"; do
  set -- $v
  n=$1; coll=$2; out=$3; bulk=$4
  tag=n${n}_${coll}_${out}_bulk${bulk}
  [ -f $O/$tag.json ] && tag=${tag}_b
  RLHEAD_RS_BULK=$bulk timeout 900 python bench.py --gpus $n $B --collective $coll --dw-output $out > $O/$tag.json 2> $O/$tag.err
  echo "$tag rc=$? $(python -c "import json; d=json.loads([l for l in open('$O/$tag.json') if l.startswith('{')][-1]); k=d['kernels']; p=d['phases_ms']; print(d['value'], d['clocks']['sm_mhz'], k['gemm_dw']['ms_total'], k['misc']['ms_total'], p['micro_batches'], p.get('min_over_ranks',{}).get('micro_batches'), p['dw_reduce'])" 2>/dev/null)"
done
