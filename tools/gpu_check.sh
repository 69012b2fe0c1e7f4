python tools/profile_chain.py C2 12
SCSF_ADAPTIVE_DEGREE=1 python tools/profile_chain.py C2 12
timeout 600 python tools/ablation.py C2 100 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('uniform', d['scsf'])"
SCSF_ADAPTIVE_DEGREE=1 timeout 600 python tools/ablation.py C2 100 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('adaptive', d['scsf'])"
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | tail -1 | head -c 150; echo
SCSF_ADAPTIVE_DEGREE=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 2>&1 | tail -1 | head -c 150; echo
SCSF_ADAPTIVE_DEGREE=1 timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_bench_config.py -x -q 2>&1 | tail -2
