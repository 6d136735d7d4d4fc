#!/bin/bash
# 1-GPU measurement set (after the dZ-from-q default): new/changed tests, the
# default bench line (all legs), cuBLAS same-shape comparison with real data,
# the HBM probe. (compute-sanitizer is closed on this pool.)
mkdir -p gpurun_out/r2f
O=gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_dz_q.py tests/test_gpu_hbm_kernels.py tests/test_gpu_parity.py tests/test_gpu_advantage.py -q -m gpu > $O/tests.log 2>&1
echo "tests_rc=$?"; tail -n 2 $O/tests.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
echo "bench_rc=$?"
python -c "import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e'], d['clocks'], d['roofline'], d['aux'].get('torch_eager_reference'))"
timeout 900 python scripts/probe.py --config qwen7b --rows 16384 --reps 3 --cublas --sustain 20 > $O/cublas_compare.json 2>&1
echo "cublas_rc=$?"; cat $O/cublas_compare.json
timeout 300 python scripts/probe_hbm.py --reps 5 > $O/probe_hbm.json 2>&1
cat $O/probe_hbm.json
