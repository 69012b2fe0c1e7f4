# usage: bash tools/gpu_check.sh  (GPU box)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_chain.py C2 6 && python tools/profile_chain.py C2 6
python tools/chain_phases.py C2 256 1 16
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_v9.csv python tools/profile_chain.py C2 6 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_C2_v9.csv | head -24
for c in 16 24; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --chains-per-gpu $c 2>&1 | tail -1 | head -c 200; echo; done
