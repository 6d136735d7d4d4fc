# 4-GPU bench: fused dW reduce-scatter (symm) vs NCCL all-reduce
for c in symm nccl; do
  extra=""; [ $c = nccl ] && extra="--no-e2e --no-aux"
  timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --collective $c $extra > gpurun_out/bench_dp4_$c.log 2>&1; echo "$c rc=$?"
  grep '^{' gpurun_out/bench_dp4_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['config']['dw_collective'], d['clocks'], d['e2e'] and d['e2e']['value'])" || tail -c 2000 gpurun_out/bench_dp4_$c.log
done
