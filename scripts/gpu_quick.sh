# quick GPU iteration: parity tests (fwd-focused) + short bench
set -x
timeout 300 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -25
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu ${BENCH_ARGS} 2>&1 | tail -3
