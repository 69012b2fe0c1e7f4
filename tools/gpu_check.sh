# usage: bash tools/gpu_check.sh  (GPU box)
timeout 300 python -m pytest tests/test_gpu_components.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3
for r in 128 512 1024; do SCSF_TN_MIN_ROWS=$r timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | tail -1 | head -c 120; echo " rows=$r"; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
