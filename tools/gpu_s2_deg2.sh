# per-column degree sweeps for C2 and C4 (the configs besides the C3 headline)
set -x
timeout 900 python tools/degree_sweep.py C2:1000:32 --m=-80,-120,-160 > gpurun_out/s2d_C2_sweep.jsonl 2> gpurun_out/s2d_C2_sweep.err
timeout 900 python tools/degree_sweep.py C4:200:32 --m=-200,-256 > gpurun_out/s2d_C4_sweep.jsonl 2> gpurun_out/s2d_C4_sweep.err
cat gpurun_out/s2d_C2_sweep.jsonl gpurun_out/s2d_C4_sweep.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['config'],d['m'],round(d['operators_per_s'],2),d['converged'],d['iterations_mean'])"
