# A/B of the cluster filter: static-parity two-step loop (lib/) vs the previous kernel (lib_ab/)
set -x
timeout 900 python -m pytest tests/test_gpu_solve.py -q -k "filter or adaptive or chains_matches" > gpurun_out/s2_ftests.log 2>&1; echo rc=$? >> gpurun_out/s2_ftests.log
tail -2 gpurun_out/s2_ftests.log
for d in 20 160; do
  for L in lib lib_ab; do
    BF_DEGREE=$d SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 300 python tools/bench_filter.py C2 C3 > gpurun_out/s2_bf_${L}_m$d.json 2>&1
  done
done
for L in lib lib_ab lib; do
  SCSF_LIB=$PWD/paper_2510_23215_b200/$L/libscsf.so timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-degree > gpurun_out/s2_bench_${L}.json 2> gpurun_out/s2_bench_${L}.err
  tail -c 300 gpurun_out/s2_bench_${L}.json | head -c 200; echo
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_pipes tools/fp64_pipes.cu && /tmp/fp64_pipes > gpurun_out/s2_fp64_pipes.txt 2>&1
cat gpurun_out/s2_fp64_pipes.txt
