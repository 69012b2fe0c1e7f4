# per-column degree margin (k_lock aims each column at tol / margin): C3 and C2 full queues
set -x
for M in 10 3 1 30; do
  SCSF_DEG_MARGIN=$M timeout 600 python tools/degree_sweep.py C3:400:32 --m=-256 > gpurun_out/s2m_C3_$M.jsonl 2> gpurun_out/s2m_C3_$M.err
  SCSF_DEG_MARGIN=$M timeout 600 python tools/degree_sweep.py C2:1000:32 --m=-80 > gpurun_out/s2m_C2_$M.jsonl 2> gpurun_out/s2m_C2_$M.err
  cat gpurun_out/s2m_C3_$M.jsonl gpurun_out/s2m_C2_$M.jsonl | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('margin $M', d['config'],d['m'],round(d['operators_per_s'],2),d['converged'],d['iterations_mean'],int(d['spmm_columns_mean']))"
done
