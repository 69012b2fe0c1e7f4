set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench_config.py tests/test_gpu_solve.py -q -m gpu -x > gpurun_out/guard_tests.log 2>&1; echo rc=$? >> gpurun_out/guard_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_guard.json 2> gpurun_out/bench_guard.err; echo rc=$? >> gpurun_out/bench_guard.err
