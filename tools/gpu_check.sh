# usage: bash tools/gpu_check.sh  (GPU box)
timeout 300 python -m pytest tests/test_gpu_solve.py -x -q -k filter 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_components.py -x -q 2>&1 | tail -3
python tools/bench_filter.py C1 C2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_chain.py C2 6 && python tools/profile_chain.py C2 6
for c in 16 32 48; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --chains-per-gpu $c 2>&1 | tail -1 | head -c 200; echo; done
