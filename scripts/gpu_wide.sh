timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout -s KILL 900 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -3
for v in "RLHEAD_WIDE=1" "RLHEAD_WIDE=0" "RLHEAD_CTA_GROUP=1"; do
  env $v timeout -s KILL 200 python scripts/probe.py --reps 3 | sed "s/^/$v /"
done
