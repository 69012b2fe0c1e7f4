# session 4 (container re-created, tree rebuilt from HEAD): bench line first, then smoke, then the GPU suite
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s4_bench_C3.json 2> gpurun_out/s4_bench_C3.err; echo bench_rc=$?
tail -c 600 gpurun_out/s4_bench_C3.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s4_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/s4_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_tests.log
tail -3 gpurun_out/s4_tests.log
