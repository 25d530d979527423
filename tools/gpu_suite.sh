# GPU test suite, then (BENCH=1) one default bench line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
if [ -n "$BENCH" ]; then timeout 600 python bench.py 2>/dev/null | tail -c 2500; fi
