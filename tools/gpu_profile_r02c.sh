set -x
timeout 600 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "cluster_variants or filter_matches" > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
for sp in 0 1; do
  SCSF_FILTER_SPLIT=$sp timeout 200 python tools/bench_filter.py C2 C3 > gpurun_out/bfsplit_$sp.json 2>&1
  SCSF_FILTER_SPLIT=$sp timeout 300 python tools/graph_ab.py C3 64 32 120 >> gpurun_out/split_ab.jsonl 2>/dev/null
  SCSF_FILTER_SPLIT=$sp timeout 300 python tools/graph_ab.py C2 1000 32 20 >> gpurun_out/split_ab.jsonl 2>/dev/null
done
# single-chain launch list (C3, 2 operators, m = 120): per-kernel device time, serialised
CMD="python tools/profile_chain.py C3 2 1 120"
timeout 300 $CMD > gpurun_out/chain_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_chain.csv $CMD > gpurun_out/ncu_chain.log 2>&1
echo chain_rc=$?
