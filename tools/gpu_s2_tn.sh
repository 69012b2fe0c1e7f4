# 128-wide TMA TN tile (SCSF_TN_WIDE=1, default) vs the 64-wide tile: parity, isolated shapes, C3 bench; C2/C4 degree sweeps
set -x
timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_solve.py -q -x -k "gemm or full_size_chain or chains_matches" > gpurun_out/s2t_tests.log 2>&1; echo rc=$? >> gpurun_out/s2t_tests.log
tail -2 gpurun_out/s2t_tests.log
grep -q "rc=0" gpurun_out/s2t_tests.log || exit 1
for W in 0 1; do SCSF_TN_WIDE=$W timeout 300 python tools/gemm_ab.py > gpurun_out/s2t_gemm_ab_$W.json 2>&1; done
python - <<'PY'
import json
for W in "01":
    try:
        d=json.load(open(f"gpurun_out/s2t_gemm_ab_{W}.json"))
        rows=d.get("rows", d)
        print(W, [(r["config"], round(r["tn_upper_us"],1), round(r["tn_full_us"],1)) for r in rows])
    except Exception as e:
        print(W, "parse", e, open(f"gpurun_out/s2t_gemm_ab_{W}.json").read()[:300])
PY
for W in 1 0 1; do
  SCSF_TN_WIDE=$W timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2t_bench_$W.json 2> gpurun_out/s2t_bench_$W.err
  python -c "import json;d=json.loads(open('gpurun_out/s2t_bench_$W.json').read().strip().splitlines()[-1]);print('wide$W', d['value'], d['converged'], d['roofline_dmma']['frac'])"
done
timeout 900 python tools/degree_sweep.py C2:1000:32 --m 30,-40,40,-60 > gpurun_out/s2t_C2_sweep.jsonl 2> gpurun_out/s2t_C2_sweep.err
timeout 900 python tools/degree_sweep.py C4:200:32 --m -200,-256 > gpurun_out/s2t_C4_sweep.jsonl 2> gpurun_out/s2t_C4_sweep.err
cat gpurun_out/s2t_C2_sweep.jsonl gpurun_out/s2t_C4_sweep.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['config'],d['m'],round(d['operators_per_s'],2),d['converged'],d['iterations_mean'])"
