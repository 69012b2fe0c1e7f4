# usage: bash tools/gpu_check.sh  (GPU box)
timeout 300 python -m pytest tests/test_gpu_solve.py -x -q -k filter 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_bench_config.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 600 python tools/ablation.py C2 200 > gpurun_out/ablation_C2.json 2>&1; cat gpurun_out/ablation_C2.json
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | tail -1 | head -c 150; echo
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
