# session 3: last check of the committed tree (GPU suite + smoke)
set -x
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/s3l_tests.log 2>&1; echo rc=$? >> gpurun_out/s3l_tests.log
tail -3 gpurun_out/s3l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3l_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s3l_smoke.log
