set -x
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python scripts/time_fwd.py t 2>&1 | tail -12
timeout 120 python scripts/trace_fwd.py 2>&1 | tail -3
