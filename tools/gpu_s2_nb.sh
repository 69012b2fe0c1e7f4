# x-neighbours by shared loads (lib_ab/, -DSCSF_NB_LDS) vs warp shuffles (lib/, default)
set -x
SCSF_LIB=$PWD/paper_2510_23215_b200/lib_ab/libscsf.so timeout 600 python -m pytest tests/test_gpu_solve.py -q -x -k "tmem_variant or filter_matches or split" > gpurun_out/s2b_tests.log 2>&1; echo rc=$? >> gpurun_out/s2b_tests.log
tail -2 gpurun_out/s2b_tests.log
for r in 1 2; do
for L in lib lib_ab; do
  BF_DEGREE=192 SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 300 python tools/bench_filter.py C2 C3 > gpurun_out/s2b_bf_${L}_$r.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/s2b_bf_${L}_$r.json'));print('$L', {k:(round(v['ms_per_filter'],3),round(v['us_per_step'],2)) for k,v in d.items()})"
done
done
