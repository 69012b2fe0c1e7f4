# C3 full queue, 32 chains, filter degree m: throughput with the split-sync filter (3 timed steps each)
set -x
for m in 160 192 224 256; do
  timeout 900 python bench.py --degree $m --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2_deg_$m.json 2> gpurun_out/s2_deg_$m.err
  python -c "import json;d=json.loads(open('gpurun_out/s2_deg_$m.json').read().strip().splitlines()[-1]);print('m=$m', d['value'], d['converged'], d['iterations_mean'], d['iterations_max'], d['roofline']['avg_launch_us'])"
done
