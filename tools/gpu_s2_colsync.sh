# per-column mbarriers in the neighbour-sync filter (lib/) vs per-step mbarriers (lib_ab/ = HEAD)
set -x
timeout 600 python -m pytest tests/test_gpu_solve.py -q -x -k "split or tmem_variant or adaptive or filter_matches" > gpurun_out/s2c_tests.log 2>&1; echo rc=$? >> gpurun_out/s2c_tests.log
tail -3 gpurun_out/s2c_tests.log
grep -q "rc=0" gpurun_out/s2c_tests.log || exit 1
for d in 20 192; do
  for L in lib lib_ab; do
    BF_DEGREE=$d SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 300 python tools/bench_filter.py C2 C3 > gpurun_out/s2c_bf_${L}_m$d.json 2>&1
  done
done
for f in gpurun_out/s2c_bf_*; do echo $f; python -c "import json;d=json.load(open('$f'));print({k:(round(v['ms_per_filter'],3),round(v['us_per_step'],2)) for k,v in d.items()})"; done
for L in lib lib_ab lib; do
  SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2c_bench_$L.json 2> gpurun_out/s2c_bench_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/s2c_bench_$L.json').read().strip().splitlines()[-1]);print('$L', d['value'], d['converged'], d['roofline']['avg_launch_us'])"
done
