# session 4: launch list of the default bench (kernel shares on the final tree), then the C2 line and the reference arm
set -x
mkdir -p gpurun_out
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/s4_launches_C3.csv python bench.py --steps 1 --warmup 1 --n-ops 32 --no-paper-degree --no-e2e --no-cpu-baseline > gpurun_out/s4_ncu.log 2>&1; echo ncu_rc=$?
timeout 400 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/s4_bench_C2.json 2> gpurun_out/s4_bench_C2.err; echo c2_rc=$?
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/s4_bench_reference.json 2> gpurun_out/s4_bench_reference.err; echo ref_rc=$?
tail -c 300 gpurun_out/s4_bench_C2.json; tail -c 300 gpurun_out/s4_bench_reference.json
