# try_wait acquire scope in the neighbour-sync filter: .cluster (lib/, HEAD) vs .cta (lib_ab/, no CCTL.IVALL per wait)
set -x
for r in 1 2; do
for L in lib lib_ab; do
  BF_DEGREE=192 SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 300 python tools/bench_filter.py C2 C3 > gpurun_out/s2a_bf_${L}_$r.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/s2a_bf_${L}_$r.json'));print('$L', {k:(round(v['ms_per_filter'],3),round(v['us_per_step'],2)) for k,v in d.items()})"
done
done
for L in lib_ab lib; do
  SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2a_bench_$L.json 2> gpurun_out/s2a_bench_$L.err
  python -c "import json;d=json.loads(open('gpurun_out/s2a_bench_$L.json').read().strip().splitlines()[-1]);print('$L', d['value'], d['converged'], d['roofline']['avg_launch_us'])"
done
