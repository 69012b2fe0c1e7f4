set -x
for u in 4 5 6 8; do SCSF_BJ_UNROLL=$u timeout 300 python tools/graph_ab.py C3 64 32 120 >> gpurun_out/unroll_ab.jsonl 2>/dev/null; done
timeout 900 python bench.py --config C2 --steps 10 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-paper-degree > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 1500 python bench.py --config C5 --n-ops 4 --steps 3 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
