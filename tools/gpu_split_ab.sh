set -x
timeout 120 python -m pytest tests/test_gpu_solve.py -q -m gpu -x -k "cluster_variants" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
for sp in 0 1; do
  SCSF_FILTER_SPLIT=$sp timeout 100 python tools/bench_filter.py C2 C3 > gpurun_out/bfsplit_$sp.json 2>&1
  SCSF_FILTER_SPLIT=$sp timeout 200 python tools/graph_ab.py C3 64 32 120 >> gpurun_out/split_ab2.jsonl 2>/dev/null
done
