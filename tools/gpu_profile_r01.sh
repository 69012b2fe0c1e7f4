set -x
python tools/profile_chain.py C2 6
for c in 8 32 64; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 2 --warmup 1 --chains-per-gpu $c > gpurun_out/bench_c$c.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python tools/profile_chain.py C2 6 > gpurun_out/ncu_launch.log 2>&1
for k in k_filter_res2d k_jacobi_x k_chol_inv k_gemm_tn2 k_gemm_nn2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 12 -c 1 -o gpurun_out/full_$k python tools/profile_chain.py C2 3 > gpurun_out/ncu_$k.log 2>&1
done
timeout 300 python tools/profile_chain.py C3 2
timeout 300 python tools/profile_chain.py C4 2
