set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full2.json 2> gpurun_out/bench_full2.err
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/bench_C2b.json 2> gpurun_out/bench_C2b.err
timeout 200 python tools/bench_filter.py C3 > gpurun_out/bf_tm.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_cl -s 2 -c 1 -o gpurun_out/prof_filter_c3_tmem python tools/bench_filter.py C3 > gpurun_out/ncu_filter_tm.log 2>&1
echo ncu_rc=$?
