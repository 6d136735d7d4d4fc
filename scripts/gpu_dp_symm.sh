# 2-GPU: fused DP dW reduce-scatter + TP symmetric-memory tests
timeout -s KILL 900 python -m pytest tests/test_gpu_tp_symm.py -q -x 2>&1 | tail -5
for args in "--config qwen7b --mb-rows 65536 --max-mb 2" "--config openvla --mb-rows 65536 --max-mb 1"; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29541 scripts/dp_check.py $args --reps 3 > gpurun_out/dp_symm.log 2>&1; echo "dp $args rc=$?"
  grep '^{' gpurun_out/dp_symm.log || tail -c 3000 gpurun_out/dp_symm.log
done
