# Final tree on 4 B200: the driver's scaling command for N=4 (defaults).
mkdir -p gpurun_out
timeout -s KILL 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_dp4_final.log 2>&1; echo "rc=$?"
grep '^{' gpurun_out/bench_dp4_final.log | tail -1 > gpurun_out/bench_dp4_final.json
python -c "import json; d=json.load(open('gpurun_out/bench_dp4_final.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_executed_frac_burst'], d['config']['lpt_load_max_over_mean'])" || tail -c 2000 gpurun_out/bench_dp4_final.log
