# final check of the committed tree: GPU suite, smoke, bench line
set -x
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/s2g_tests.log 2>&1; echo rc=$? >> gpurun_out/s2g_tests.log
tail -3 gpurun_out/s2g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2g_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s2g_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s2g_bench.json 2> gpurun_out/s2g_bench.err
python -c "import json;d=json.loads(open('gpurun_out/s2g_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu']['frac'], d['roofline_dmma']['frac'], d['converged'], d['iterations_mean'], d['clocks'], d['gpu_launches'])"
