# 2-GPU: vocab-parallel dL/dH sum over NVLink peer memory vs NCCL
nvidia-smi topo -m | head -4
timeout -s KILL 300 python -m pytest tests/test_gpu_vocab_parallel.py -q -x 2>&1 | tail -4
for cfg in "qwen1.5b 4096" "qwen7b 16384" "qwen7b 65536"; do
  set -- $cfg
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 scripts/tp_check.py --config $1 --rows $2 \
    --reps 3 > gpurun_out/tp_symm_$1_$2.log 2>&1; echo "tp $1 $2 rc=$?"
  grep '^{' gpurun_out/tp_symm_$1_$2.log || tail -c 3000 gpurun_out/tp_symm_$1_$2.log
done
