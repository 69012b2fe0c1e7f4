set -x
timeout 600 python -m pytest tests/test_gpu_solve.py -q -m gpu -x -k "filter_matches or bad_arguments or tmem" > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
timeout 900 python tools/degree_sweep.py C3:400:32 --m 120,144,160,192 > gpurun_out/sweep_hi.jsonl 2>/dev/null
timeout 600 python tools/degree_sweep.py C4:200:32 --m 80,120 >> gpurun_out/sweep_hi.jsonl 2>/dev/null
timeout 300 python tools/degree_sweep.py C5:4:4 --m 80,120 >> gpurun_out/sweep_hi.jsonl 2>/dev/null
