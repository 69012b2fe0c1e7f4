# session 4: the C4 line on the rebuilt tree
mkdir -p gpurun_out
timeout 420 python bench.py --config C4 --steps 3 --warmup 3 --no-paper-degree --no-cpu-baseline > gpurun_out/s4_bench_C4.json 2> gpurun_out/s4_bench_C4.err; echo c4_rc=$?
tail -c 400 gpurun_out/s4_bench_C4.json
