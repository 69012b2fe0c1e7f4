set -x
# ncu segfaulted (exit 11) on the graph-replayed 32-chain bench (the same command exits 0 without ncu);
# the launch list is taken with SCSF_GRAPHS=0 (the same kernels, launched eagerly)
BENCH="python bench.py --steps 1 --warmup 1 --n-ops 64 --no-e2e --no-cpu-baseline --no-paper-degree --roofline-ops 2"
SCSF_GRAPHS=0 timeout 600 $BENCH > gpurun_out/bench_small_eager.json 2> gpurun_out/bench_small_eager.err && \
SCSF_GRAPHS=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 80000 -c 8000 --csv --log-file gpurun_out/launches_c3.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
echo launch_rc=$?
