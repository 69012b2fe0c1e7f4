set -x
timeout 300 python -m pytest tests/test_gpu_solve.py -q -m gpu -x -k "zmarch or filter_matches" > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
SCSF_Z3=0 timeout 120 python tools/bench_filter.py C4 > gpurun_out/bfz3_off.json 2>&1
for zc in 4 5 8 10 20 40; do SCSF_Z3_ZC=$zc timeout 120 python tools/bench_filter.py C4 > gpurun_out/bfz3_$zc.json 2>&1; done
SCSF_Z3=0 timeout 300 python tools/degree_sweep.py C4:64:32 --m 80 > gpurun_out/z3_sweep.jsonl 2>/dev/null
timeout 300 python tools/degree_sweep.py C4:64:32 --m 80 >> gpurun_out/z3_sweep.jsonl 2>/dev/null
timeout 300 python -m pytest tests/test_gpu_components.py -q -m gpu -x -k "gemm_nn" > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
for v in 0 1; do SCSF_NN4=$v timeout 200 python tools/gemm_ab.py > gpurun_out/gemm_nn4_$v.json 2>/dev/null; done
for v in 0 1; do SCSF_NN4=$v timeout 300 python tools/degree_sweep.py C5:4:4 --m 80 >> gpurun_out/nn4_c5.jsonl 2>/dev/null; done
