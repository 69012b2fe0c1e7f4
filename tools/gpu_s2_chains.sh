# concurrent chains per GPU on the full C3 queue (per-column degrees <= 256)
set -x
for C in 16 24 32 48 64; do
  timeout 600 python tools/degree_sweep.py C3:400:$C --m=-256 > gpurun_out/s2k_C3_$C.jsonl 2> gpurun_out/s2k_C3_$C.err
  python -c "
import json
for l in open('gpurun_out/s2k_C3_$C.jsonl'):
  d=json.loads(l); print('chains $C', round(d['operators_per_s'],2), d['converged'], d['iterations_mean'], d.get('iterations_cold_mean'))"
done
