# v6 kernels on the other BASELINE configs (1 GPU): Qwen-1.5B head, OpenVLA head.
mkdir -p gpurun_out
for cfg in qwen1.5b openvla; do
  timeout -s KILL 1200 python bench.py --config $cfg > gpurun_out/bench_v6_$cfg.json 2> gpurun_out/bench_v6_$cfg.err; echo "$cfg rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/bench_v6_$cfg.json')); print('$cfg', d['value'], d['ms_per_step'], d['clocks'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_executed_frac_burst'], d['cpu_baseline']['value'])" || tail -c 1500 gpurun_out/bench_v6_$cfg.err
done
