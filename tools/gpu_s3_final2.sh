# session 3, final check of the committed tree (trimmed filter clusters on): cluster-slot probe,
# full GPU suite, smoke, C3 bench line
set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_slots tools/cluster_slots.cu && /tmp/cluster_slots > gpurun_out/s3f_cluster_slots.json
cat gpurun_out/s3f_cluster_slots.json
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/s3f_tests.log 2>&1; echo rc=$? >> gpurun_out/s3f_tests.log
tail -3 gpurun_out/s3f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3f_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/s3f_smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s3f_bench.json 2> gpurun_out/s3f_bench.err
python -c "import json;d=json.loads(open('gpurun_out/s3f_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu']['frac'], d['roofline_dmma']['frac'], d['converged'], d['iterations_mean'], d['clocks'], d['gpu_launches'])"
