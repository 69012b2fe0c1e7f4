set -x
timeout 180 python -m pytest tests/test_gpu_solve.py -q -m gpu -x -k "tmem_variant" > gpurun_out/t16.log 2>&1; echo rc=$? >> gpurun_out/t16.log
grep -q "passed" gpurun_out/t16.log || exit 0
for v in 0 1; do SCSF_FILTER_TMEM=$v timeout 120 python tools/bench_filter.py C2 C3 > gpurun_out/bftm_$v.json 2>&1; done
for v in 0 1; do SCSF_FILTER_TMEM=$v timeout 300 python tools/graph_ab.py C3 64 32 120 >> gpurun_out/tm_ab.jsonl 2>/dev/null; SCSF_FILTER_TMEM=$v timeout 300 python tools/graph_ab.py C2 1000 32 20 >> gpurun_out/tm_ab.jsonl 2>/dev/null; done
