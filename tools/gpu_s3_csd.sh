# session 3: smallest-fitting filter cluster (SCSF_FILTER_CS_DOUBLE=0: C2 on 4-CTA clusters, 33 co-resident)
# against the doubled 8-CTA clusters (15 co-resident): parity, then the C2 / C1 bench A/B
set -x
mkdir -p gpurun_out
SCSF_FILTER_CS_DOUBLE=0 timeout 900 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "filter" > gpurun_out/s3c_tests.log 2>&1; echo rc=$? >> gpurun_out/s3c_tests.log
tail -3 gpurun_out/s3c_tests.log
grep -q "rc=0" gpurun_out/s3c_tests.log || exit 1
for t in 1 0 1 0; do SCSF_FILTER_CS_DOUBLE=$t timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s3c_C2_$t.json 2> gpurun_out/s3c_C2_$t.err; python -c "import json;d=json.loads(open('gpurun_out/s3c_C2_$t.json').read().strip().splitlines()[-1]);print('C2 csd=$t', d['value'], d['converged'], d['clocks'])"; done
