# session 2 of round 2: confirm the restored tree on a B200 (GPU suite + default bench line)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/s2_tests.log 2>&1; echo rc=$? >> gpurun_out/s2_tests.log
tail -3 gpurun_out/s2_tests.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
echo bench_rc=$?
tail -c 600 gpurun_out/s2_bench.json
