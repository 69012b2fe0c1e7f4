cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_components.py -q -m gpu -x -k "gemm" > gpurun_out/nn_tests.log 2>&1; echo rc=$? >> gpurun_out/nn_tests.log
SCSF_NN_TMA=0 timeout 300 python tools/nn_ab.py > gpurun_out/nn_ab0.json 2>gpurun_out/nn_ab0.err
SCSF_NN_TMA=1 timeout 300 python tools/nn_ab.py > gpurun_out/nn_ab1.json 2>gpurun_out/nn_ab1.err
SCSF_TRACE=1 timeout 600 python tools/diag_degree.py C3 400 32 256 > gpurun_out/diag256.json 2> gpurun_out/diag256.trace
