# Multi-GPU tests (2 B200) on the current kernels.
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest -q -x -m gpu tests/test_gpu_tp_symm.py tests/test_gpu_vocab_parallel.py tests/test_gpu_dw_reduce_scatter.py > gpurun_out/gpu_tests_2gpu.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_2gpu.log
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 > gpurun_out/bench_dp2_v5.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_dp2_v5.log | tail -1 > gpurun_out/bench_dp2_v5.json
python -c "import json; d=json.load(open('gpurun_out/bench_dp2_v5.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'])" || tail -c 1500 gpurun_out/bench_dp2_v5.log
