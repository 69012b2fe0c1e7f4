# bench lines of C2 and C4 at their per-column degrees, C5 row partition degree probe
set -x
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 > gpurun_out/s2l_C2.json 2> gpurun_out/s2l_C2.err
python -c "import json;d=json.loads(open('gpurun_out/s2l_C2.json').read().strip().splitlines()[-1]);print('C2', d['value'], d['e2e']['value'] if d.get('e2e') else None, d['converged'], d.get('paper_degree',{}).get('value'))"
timeout 1200 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/s2l_C4.json 2> gpurun_out/s2l_C4.err
python -c "import json;d=json.loads(open('gpurun_out/s2l_C4.json').read().strip().splitlines()[-1]);print('C4', d['value'], d['e2e']['value'] if d.get('e2e') else None, d['converged'], d['roofline']['frac'], d.get('paper_degree',{}).get('value'))"
for m in 80 -120 -160; do
  timeout 900 python bench.py --config C5 --degree=$m --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s2l_C5_$m.json 2> gpurun_out/s2l_C5_$m.err
  python -c "import json;d=json.loads(open('gpurun_out/s2l_C5_$m.json').read().strip().splitlines()[-1]);print('C5 $m', d['value'], d.get('converged'))"
done
