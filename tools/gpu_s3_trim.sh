# session 3: trimmed filter clusters (SCSF_FILTER_TRIM) -- parity first, then isolated and in-step A/B
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py -q -m gpu -k "filter or split or chains" > gpurun_out/s3t_tests.log 2>&1; echo rc=$? >> gpurun_out/s3t_tests.log
tail -3 gpurun_out/s3t_tests.log
grep -q "rc=0" gpurun_out/s3t_tests.log || exit 1
for t in 0 1 0 1; do SCSF_FILTER_TRIM=$t BF_DEGREE=192 timeout 300 python tools/bench_filter.py C3 > gpurun_out/s3t_bf_$t.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/s3t_bf_$t.json'));print('trim=$t', d['C3']['ms_per_filter'])"; done
for t in 1 0 1; do SCSF_FILTER_TRIM=$t timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s3t_bench_$t.json 2> gpurun_out/s3t_bench_$t.err; python -c "import json;d=json.loads(open('gpurun_out/s3t_bench_$t.json').read().strip().splitlines()[-1]);print('trim=$t', d['value'], d['converged'], d['clocks'])"; done
