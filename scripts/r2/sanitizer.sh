#!/bin/bash
# compute-sanitizer over the smoke (tcgen05 bf16 + fp32 SIMT head) and the
# single-GPU emulated fused dW reduce-scatter: racecheck (shared-memory
# hazards), synccheck (barrier misuse), memcheck (out-of-bounds / misaligned).
mkdir -p gpurun_out/san
O=gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 99 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?"
  timeout 1200 $CS --tool $tool --error-exitcode 99 python -m pytest -q -x tests/test_gpu_dw_reduce_scatter.py > $O/dwrs_$tool.log 2>&1
  echo "dw_reduce_scatter $tool rc=$?"
done
timeout 900 python scripts/probe.py --config qwen7b --rows 16384 --reps 3 --cublas --sustain 20 > $O/../cublas_compare.json 2>&1
echo "cublas rc=$?"
