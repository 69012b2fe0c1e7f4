# per-column degrees through the row partition's slab step: parity (loopback 1/2/3 slabs) and C5 bench
set -x
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_c5.py -q -x > gpurun_out/s2c5_tests.log 2>&1; echo rc=$? >> gpurun_out/s2c5_tests.log
tail -2 gpurun_out/s2c5_tests.log
grep -q "rc=0" gpurun_out/s2c5_tests.log || exit 1
for m in -160 -256 -120; do
  timeout 900 python bench.py --config C5 --degree=$m --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s2c5_$m.json 2> gpurun_out/s2c5_$m.err
  python -c "import json;d=json.loads(open('gpurun_out/s2c5_$m.json').read().strip().splitlines()[-1]);print('C5 $m', d['value'], d.get('converged'), d.get('iterations_mean'))"
done
