timeout -s KILL 200 python scripts/probe.py --reps 3
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
