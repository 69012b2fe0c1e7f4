"""Key metrics of `ncu --set full` reports as JSON (one object per report).
  python tools/ncu_summary.py gpurun_out/a.ncu-rep [...] > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]


def summarise(path):
    """One summary per profiled launch of the report (a list when there are several)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = [summarise_row(rows[0], rows[1], v) for v in rows[2:]]
    return res[0] if len(res) == 1 else res


def summarise_row(hdr, units, vals):
    res = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            res[k] = f"{vals[i]} {units[i]}".strip()
    stalls = []
    for i, k in enumerate(hdr):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), k.split("stalled_")[1].split("_per_")[0]))
            except ValueError:
                pass
    res["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:5]}
    return res


if __name__ == "__main__":
    print(json.dumps({p.split("/")[-1]: summarise(p) for p in sys.argv[1:]}, indent=1))
