set -x
BENCH="python bench.py --steps 1 --warmup 1 --n-ops 64 --no-e2e --no-cpu-baseline --no-paper-degree --roofline-ops 2"
timeout 600 $BENCH > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 60000 -c 6000 --csv --log-file gpurun_out/launches_c3.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
timeout 200 python tools/bench_filter.py C3 > gpurun_out/bf_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_cl -s 2 -c 1 -o gpurun_out/prof_filter_c3 python tools/bench_filter.py C3 > gpurun_out/ncu_filter.log 2>&1
echo filt_rc=$?
timeout 200 python tools/prof_kernels.py C4 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_stencil_v4g|k_gemm_tn_tma" -s 5 -c 4 -o gpurun_out/prof_c4 python tools/prof_kernels.py C4 > gpurun_out/ncu_c4.log 2>&1
echo c4_rc=$?
