# mbarrier neighbour sync (SCSF_FILTER_SPLIT=2, st.async ghost pushes) vs split arrive/wait (=1): parity, then A/B
set -x
timeout 600 python -m pytest tests/test_gpu_solve.py -q -x -k "split or tmem_variant" > gpurun_out/s2n_tests.log 2>&1; echo rc=$? >> gpurun_out/s2n_tests.log
tail -3 gpurun_out/s2n_tests.log
grep -q "rc=0" gpurun_out/s2n_tests.log || exit 1
for d in 20 160; do
  for S in 1 2; do
    SCSF_FILTER_SPLIT=$S BF_DEGREE=$d timeout 300 python tools/bench_filter.py C2 C3 > gpurun_out/s2n_bf_split${S}_m$d.json 2>&1
  done
done
for f in gpurun_out/s2n_bf_*; do echo $f; python -c "import json;d=json.load(open('$f'));print({k:(round(v['ms_per_filter'],3),round(v['us_per_step'],2)) for k,v in d.items()})"; done
for S in 2 1 2; do
  SCSF_FILTER_SPLIT=$S timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2n_bench_split$S.json 2> gpurun_out/s2n_bench_split$S.err
  python -c "import json;d=json.loads(open('gpurun_out/s2n_bench_split$S.json').read().strip().splitlines()[-1]);print('split$S', d['value'], d['converged'], d['roofline']['avg_launch_us'])"
done
