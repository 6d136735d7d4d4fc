# Restored tree on 2 B200: multi-GPU tests, the driver's N=2 bench command, cpu_baseline leg timing.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest -q -x -m gpu tests/test_gpu_tp_symm.py tests/test_gpu_vocab_parallel.py tests/test_gpu_dw_reduce_scatter.py > gpurun_out/gpu_tests_2gpu_restored.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_2gpu_restored.log
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_dp2_restored.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_dp2_restored.log | tail -1 > gpurun_out/bench_dp2_restored.json
python -c "import json; d=json.load(open('gpurun_out/bench_dp2_restored.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['frac'])" || tail -c 1500 gpurun_out/bench_dp2_restored.log
timeout -s KILL 300 python -c "
import bench
from workload import CONFIGS, make_layout
cfg = CONFIGS['qwen7b']; lay = make_layout(cfg, seed=0)
print(bench.cpu_baseline(cfg, lay, 0, 1536))" > gpurun_out/cpu_baseline_1536.log 2>&1; echo "cpu rc=$?"; tail -2 gpurun_out/cpu_baseline_1536.log
