# GPU suite + bench line with per-column degrees (-256)
set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/s2y_tests.log 2>&1; echo rc=$? >> gpurun_out/s2y_tests.log
tail -3 gpurun_out/s2y_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s2y_bench.json 2> gpurun_out/s2y_bench.err
echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/s2y_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu']['frac'], d['roofline_dmma']['frac'], d['converged'], d['iterations_mean'], d['clocks'])"
