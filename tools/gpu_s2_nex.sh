# extra-column sweep at the bench degree (C3 full queue, 32 chains) + the bench launch list (one chain, 2 operators)
set -x
timeout 900 python tools/degree_sweep.py C3:400:32 --m 192 --nex 24,32,40,56,72 > gpurun_out/s2x_nex.jsonl 2> gpurun_out/s2x_nex.err
cat gpurun_out/s2x_nex.jsonl
CMD="python bench.py --steps 1 --warmup 1 --n-ops 2 --chains-per-gpu 1 --no-e2e --no-cpu-baseline --no-paper-degree --roofline-ops 1"
timeout 300 $CMD > gpurun_out/s2x_bench_1chain.json 2> gpurun_out/s2x_bench_1chain.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2x_launches_c3_1chain.csv $CMD > gpurun_out/s2x_ncu_1chain.log 2>&1
echo launchlist_rc=$?
gzip -f gpurun_out/s2x_launches_c3_1chain.csv; ls -la gpurun_out/s2x_launches_c3_1chain.csv.gz
