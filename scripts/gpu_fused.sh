timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for v in "RLHEAD_FUSED_BWD=1" "RLHEAD_FUSED_BWD=0" "RLHEAD_FUSED_BWD=1"; do
  env $v timeout -s KILL 300 python scripts/probe.py --reps 4 --sustain 15 | sed "s/^/$v /"
done
