# Multi-GPU tests (2 B200) on the current kernels.
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest -q -x -m gpu tests/test_gpu_tp_symm.py tests/test_gpu_vocab_parallel.py tests/test_gpu_dw_reduce_scatter.py > gpurun_out/gpu_tests_2gpu.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_2gpu.log
