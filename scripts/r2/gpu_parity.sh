#!/bin/bash
# Round-2 parity run: new full-size oracle + edge-branch tests, then the whole GPU suite.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_start.csv 2>&1
timeout 1500 python -m pytest tests/test_gpu_edge_branches.py tests/test_gpu_fullsize.py -q -m gpu -x --durations=20 > gpurun_out/r2_parity_new.log 2>&1
echo "new_rc=$?"
timeout 1500 python -m pytest tests -q -m gpu --durations=15 --ignore=tests/test_gpu_fullsize.py --ignore=tests/test_gpu_edge_branches.py > gpurun_out/r2_gpu_suite.log 2>&1
echo "suite_rc=$?"
tail -n 3 gpurun_out/r2_parity_new.log; tail -n 3 gpurun_out/r2_gpu_suite.log
