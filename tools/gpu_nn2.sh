cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_components.py -q -m gpu -x -k "gemm" > gpurun_out/nn_tests.log 2>&1; echo rc=$? >> gpurun_out/nn_tests.log
timeout 300 python tools/nn_ab.py > gpurun_out/nn_ab1.json 2>gpurun_out/nn_ab1.err
SCSF_NNT_MIN_K=64 timeout 300 python tools/nn_ab.py > gpurun_out/nn_ab64.json 2>gpurun_out/nn_ab64.err
SCSF_TRACE=1 timeout 600 python tools/diag_degree.py C3 400 32 256 > gpurun_out/diag256b.json 2> gpurun_out/diag256b.trace
timeout 1500 python -m pytest tests/test_gpu_bench_config.py -q -m gpu -x > gpurun_out/guard_tests.log 2>&1; echo rc=$? >> gpurun_out/guard_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_nnt.json 2> gpurun_out/bench_nnt.err; echo rc=$? >> gpurun_out/bench_nnt.err
