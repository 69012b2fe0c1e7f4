# per-column adaptive degree (f2, degree < 0) and fewer extra columns at the bench's degree, full C3 queue
set -x
timeout 1500 python tools/degree_sweep.py C3:400:32 --m 192,-192,-256 --nex 24,40 > gpurun_out/s2f_sweep.jsonl 2> gpurun_out/s2f_sweep.err
cat gpurun_out/s2f_sweep.jsonl
