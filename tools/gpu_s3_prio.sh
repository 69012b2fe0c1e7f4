# session 3: cluster filter at the greatest execution priority (SCSF_FILTER_PRIO=1) vs the stream's
set -x
mkdir -p gpurun_out
SCSF_FILTER_PRIO=1 timeout 900 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "filter or chains" > gpurun_out/s3p_tests.log 2>&1; echo rc=$? >> gpurun_out/s3p_tests.log
tail -3 gpurun_out/s3p_tests.log
grep -q "rc=0" gpurun_out/s3p_tests.log || exit 1
for t in 1 0 1 0; do SCSF_FILTER_PRIO=$t timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s3p_C3_$t.json 2> gpurun_out/s3p_C3_$t.err; python -c "import json;d=json.loads(open('gpurun_out/s3p_C3_$t.json').read().strip().splitlines()[-1]);print('C3 prio=$t', d['value'], d['converged'], d['clocks'])"; done
for t in 1 0; do SCSF_FILTER_PRIO=$t timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s3p_C2_$t.json 2> gpurun_out/s3p_C2_$t.err; python -c "import json;d=json.loads(open('gpurun_out/s3p_C2_$t.json').read().strip().splitlines()[-1]);print('C2 prio=$t', d['value'], d['converged'], d['clocks'])"; done
