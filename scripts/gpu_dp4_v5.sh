# 4 B200, v5 kernels: Qwen-7B headline config (strong scaling of the 5.6M-token
# mini-batch, fused dW reduce-scatter), Qwen-32B head (configs[4], 19.4M tokens),
# OpenVLA head (the small-per-rank case).
mkdir -p gpurun_out
P=29561
for args in "qwen7b" "qwen32b --no-e2e --steps 2" "openvla"; do
  set -- $args; cfg=$1; shift
  timeout -s KILL 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config $cfg "$@" > gpurun_out/bench_dp4_v5_$cfg.log 2>&1; echo "$cfg rc=$?"
  P=$((P+1))
  grep '^{' gpurun_out/bench_dp4_v5_$cfg.log | tail -1 > gpurun_out/bench_dp4_v5_$cfg.json
  python -c "import json; d=json.load(open('gpurun_out/bench_dp4_v5_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['config']['dw_collective'], d['clocks'], d['e2e'] and d['e2e']['value'])" || tail -c 2000 gpurun_out/bench_dp4_v5_$cfg.log
done
