# GPU suite + bench line + ncu of the neighbour-sync filter + per-kind DGEMM profile
set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/s2w_tests.log 2>&1; echo rc=$? >> gpurun_out/s2w_tests.log
tail -3 gpurun_out/s2w_tests.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/s2w_bench.json 2> gpurun_out/s2w_bench.err
echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/s2w_bench.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline_alu']['frac'], d['roofline_dmma']['frac'], d['converged'], d['clocks'])"
BF_DEGREE=192 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_cl -s 2 -c 1 -o gpurun_out/s2w_filter_c3 python tools/bench_filter.py C3 > gpurun_out/s2w_ncu.log 2>&1
echo ncu_rc=$?
python tools/ncu_summary.py gpurun_out/s2w_filter_c3.ncu-rep > gpurun_out/s2w_ncu_summary.json 2>&1; grep -A7 "top_stalls\|gpu__time" gpurun_out/s2w_ncu_summary.json | head -12
SCSF_GEMM_PROFILE=1 timeout 300 python tools/gemm_profile.py C3 8 192 > gpurun_out/s2w_gp.out 2> gpurun_out/s2w_gp.err; python tools/gemm_profile.py --parse gpurun_out/s2w_gp.err > gpurun_out/s2w_gemm_kinds.json; cat gpurun_out/s2w_gemm_kinds.json
