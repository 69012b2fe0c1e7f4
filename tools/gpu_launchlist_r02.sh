set -x
# The bench with one chain per GPU (ncu serialises every launch; with 32 threads capturing and
# replaying graphs it did not finish / segfaulted): 8 operators of C3, m = 120, graphs on
CMD="python bench.py --steps 1 --warmup 1 --n-ops 8 --chains-per-gpu 1 --no-e2e --no-cpu-baseline --no-paper-degree --roofline-ops 1"
timeout 600 $CMD > gpurun_out/bench_1chain.json 2> gpurun_out/bench_1chain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_1chain.csv $CMD > gpurun_out/ncu_1chain.log 2>&1
echo rc=$?
