set -x
for v in 0 1 2; do SCSF_V4S=$v timeout 120 python tools/bench_filter.py C4 > gpurun_out/bfv4s_$v.json 2>&1; done
SCSF_V4S=1 timeout 300 python -m pytest tests/test_gpu_solve.py -q -m gpu -x -k "filter_matches and C4" > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
