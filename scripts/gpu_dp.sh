N=$1
nvidia-smi topo -m | head -5
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/bench_dp$N.log 2>&1; echo "rc=$?"
tail -c 2500 gpurun_out/bench_dp$N.log
