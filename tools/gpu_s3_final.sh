# session 3 of round 2: full GPU suite, smoke and the C3 bench line on the committed tree
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3_gpu.txt 2>&1
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/s3_tests.log 2>&1; echo rc=$? >> gpurun_out/s3_tests.log
tail -3 gpurun_out/s3_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s3_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
python -c "import json;d=json.loads(open('gpurun_out/s3_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu']['frac'], d['roofline_dmma']['frac'], d['converged'], d['iterations_mean'], d['clocks'], d['gpu_launches'])"
