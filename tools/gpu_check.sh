# usage: bash tools/gpu_check.sh  (GPU box)
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_chain.py C2 6 && python tools/profile_chain.py C2 6
python tools/chain_phases.py C2 256 1 8 16 32
