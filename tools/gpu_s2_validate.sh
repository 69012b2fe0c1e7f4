# session 2 of round 2: GPU suite, bench line and ncu of the filter after the split-sync / static-parity change
set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/s2v_tests.log 2>&1; echo rc=$? >> gpurun_out/s2v_tests.log
tail -3 gpurun_out/s2v_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s2v_bench.json 2> gpurun_out/s2v_bench.err
echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/s2v_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu'], d['converged'])"
BF_DEGREE=160 timeout 200 python tools/bench_filter.py C3 > gpurun_out/s2v_bf.json 2>&1 && \
BF_DEGREE=160 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_cl -s 2 -c 1 -o gpurun_out/s2v_filter_c3 python tools/bench_filter.py C3 > gpurun_out/s2v_ncu.log 2>&1
echo ncu_rc=$?
python tools/ncu_summary.py gpurun_out/s2v_filter_c3.ncu-rep > gpurun_out/s2v_ncu_summary.json 2>&1; head -40 gpurun_out/s2v_ncu_summary.json
