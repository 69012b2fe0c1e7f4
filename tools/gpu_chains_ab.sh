set -x
for c in 24 32 48 64; do timeout 400 python tools/degree_sweep.py C3:400:$c --m 120 >> gpurun_out/chains_ab.jsonl 2>/dev/null; done
for inn in 1 2; do SCSF_BJ_INNER=$inn timeout 300 python tools/graph_ab.py C3 8 1 120 >> gpurun_out/inner_ab.jsonl 2>/dev/null; SCSF_BJ_INNER=$inn timeout 300 python tools/graph_ab.py C3 64 32 120 >> gpurun_out/inner_ab.jsonl 2>/dev/null; done
