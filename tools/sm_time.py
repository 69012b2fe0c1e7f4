"""SM-time breakdown of an ncu launch list (`--metrics gpu__time_duration.sum`).

With many concurrent chains the GPU is full, so throughput is set by SM-time
(duration x SMs a launch occupies), not by the serialised kernel time.  The SM
footprint of a launch is min(grid, 148 x resident CTAs per SM) / resident CTAs
per SM, with resident CTAs per SM taken from each kernel's occupancy limit
(threads, registers, shared memory) as compiled.

  python tools/sm_time.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

# resident CTAs per SM (from ptxas register / shared-memory use and block size)
CTAS_PER_SM = {
    "k_filter_cl": 1, "k_filter_rp": 1, "k_gemm_nn3": 1, "k_jacobi_g": 1, "k_jacobi_z": 1, "k_chol_reg": 1, "k_gemm_nn2": 2, "k_gemm_tn2": 3,
    "k_reduce_partials": 8, "k_stencil_v4": 8, "k_resid": 4, "k_lock": 32, "k_gather_sign": 8,
}


def main(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        full = r[ki]
        name = full.split("(")[0].replace("void ", "").replace("scsf::", "").split("<")[0].strip()
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        grid = 1
        if gi is not None:
            g = r[gi].strip("()").split(",")
            grid = 1
            for x in g:
                grid *= int(x)
        per = CTAS_PER_SM.get(name, 4)
        sms = min(148.0, grid / per)
        a = agg[name]
        a[0] += 1
        a[1] += us
        a[2] += us * sms
    tot_t = sum(v[1] for v in agg.values())
    tot_s = sum(v[2] for v in agg.values())
    print(f"{'kernel':24s} {'launches':>8s} {'kernel us':>11s} {'share':>6s} {'SM-ms':>9s} {'SM share':>8s}")
    for k, (c, t, s) in sorted(agg.items(), key=lambda x: -x[1][2]):
        print(f"{k:24s} {c:8d} {t:11.0f} {100 * t / tot_t:5.1f}% {s / 1e3:9.1f} {100 * s / tot_s:7.1f}%")
    print(f"{'TOTAL':24s} {sum(v[0] for v in agg.values()):8d} {tot_t:11.0f}        {tot_s / 1e3:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
