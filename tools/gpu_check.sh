# usage: bash tools/gpu_check.sh  (GPU box): parity suite, chain timing, filter bench, launch list, bench
timeout 300 python -m pytest tests/test_gpu_solve.py -x -q -k "filter" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/profile_chain.py C2 6 && python tools/profile_chain.py C2 6
python tools/bench_filter.py C1 C2
python tools/bench_components.py 2>&1 | head -8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2_v6.csv python tools/profile_chain.py C2 6 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_C2_v6.csv | head -16
for c in 16 32; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --chains-per-gpu $c 2>&1 | tail -1 | head -c 200; echo; done
