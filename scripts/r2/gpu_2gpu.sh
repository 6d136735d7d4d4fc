#!/bin/bash
# 2-GPU checks: multi-GPU tests (vocab-parallel, DP dW modes, DP step vs the
# oracle), the bench's own --gpus 2 relaunch (Qwen-7B and OpenVLA heads) with
# per-phase times, and the 1-GPU OpenVLA line on the same box for scaling.
mkdir -p gpurun_out/r2_2gpu
O=gpurun_out/r2_2gpu
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_tp_symm.py -q -m gpu --durations=10 > $O/tests_2gpu.log 2>&1
echo "tests_rc=$?"; tail -n 3 $O/tests_2gpu.log
timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_qwen7b_dp2.json 2> $O/bench_qwen7b_dp2.err
echo "bench7b_rc=$?"
for n in 1 2; do
  timeout 900 python bench.py --gpus $n --config openvla --steps 10 --warmup 3 --no-cpu-baseline --phases > $O/bench_openvla_dp$n.json 2> $O/bench_openvla_dp$n.err
  echo "openvla_dp$n rc=$?"
done
python - <<'PY'
import json
for f in ["bench_qwen7b_dp2", "bench_openvla_dp1", "bench_openvla_dp2"]:
    try:
        d = json.load(open(f"gpurun_out/r2_2gpu/{f}.json"))
        print(f, d["n_gpus"], d.get("gpus_active"), d["value"], d["clocks"]["sm_mhz"], d.get("phases_ms"))
    except Exception as e:
        print(f, "ERR", e)
PY
