# other configs after the session-2 filter changes: C2 (cluster filter, 8-CTA), C4 (3-D streaming), C5 (row partition, 1 GPU)
set -x
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --no-paper-degree > gpurun_out/s2z_C2.json 2> gpurun_out/s2z_C2.err
timeout 900 python tools/degree_sweep.py C4:200:32 --m 80,-80,-120,-160 > gpurun_out/s2z_C4_sweep.jsonl 2> gpurun_out/s2z_C4_sweep.err
cat gpurun_out/s2z_C4_sweep.jsonl
timeout 900 python tools/degree_sweep.py C2:1000:32 --m 20,-20,-30 > gpurun_out/s2z_C2_sweep.jsonl 2> gpurun_out/s2z_C2_sweep.err
cat gpurun_out/s2z_C2_sweep.jsonl
python -c "import json;d=json.loads(open('gpurun_out/s2z_C2.json').read().strip().splitlines()[-1]);print('C2', d['value'], d['e2e']['value'] if d.get('e2e') else None, d['roofline']['frac'], d['converged'])"
