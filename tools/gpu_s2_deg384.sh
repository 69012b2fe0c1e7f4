# FP_MAX_DEGREE 384: argument checks, filter parity at high degree, C3 / C5 per-column degree sweeps
set -x
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x -k "bad_arguments or filter_matches or tmem_variant or split or adaptive" > gpurun_out/s2h_tests.log 2>&1; echo rc=$? >> gpurun_out/s2h_tests.log
tail -2 gpurun_out/s2h_tests.log
grep -q "rc=0" gpurun_out/s2h_tests.log || exit 1
timeout 1200 python tools/degree_sweep.py C3:400:32 --m=-256,-320,-384 > gpurun_out/s2h_C3.jsonl 2> gpurun_out/s2h_C3.err
for m in -256 -384; do
  timeout 900 python bench.py --config C5 --degree=$m --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s2h_C5_$m.json 2> gpurun_out/s2h_C5_$m.err
  python -c "import json;d=json.loads(open('gpurun_out/s2h_C5_$m.json').read().strip().splitlines()[-1]);print('C5 $m', d['value'], d.get('converged'))"
done
cat gpurun_out/s2h_C3.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['config'],d['m'],round(d['operators_per_s'],2),d['converged'],d['iterations_mean'])"
