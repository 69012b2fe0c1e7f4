timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | tail -1 | head -c 150; echo
