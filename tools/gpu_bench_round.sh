# Round-end style measurement on the GPU box: bench line, reference arm, launch list, ncu captures.
set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -c 3000 gpurun_out/bench_full.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 1500 gpurun_out/bench_ref.json
python bench.py --steps 1 --warmup 1 --n-ops 96 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_small.csv python bench.py --steps 1 --warmup 1 --n-ops 96 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_small.log 2>&1
python tools/launch_summary.py gpurun_out/launches_bench_small.csv | head -30
python tools/profile_chain.py C2 3 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_filter_cl --launch-skip 3 -c 1 -o gpurun_out/full16_filter_cl python tools/profile_chain.py C2 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_nn2 --launch-skip 40 -c 1 -o gpurun_out/full16_nn2 python tools/profile_chain.py C2 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_jacobi_g --launch-skip 5 -c 1 -o gpurun_out/full16_jacobi_g python tools/profile_chain.py C2 3 > /dev/null 2>&1
ls gpurun_out
