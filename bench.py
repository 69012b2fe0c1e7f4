#!/usr/bin/env python
"""bench.py — SCSF hot path on B200: truncated-FFT sort + warm-started ChFSI.

One step = one pass of the whole hot path over one batch: scsf_sort over the
global queue (Alg. 2; every rank computes the same permutation) + the solve of
this rank's contiguous share of the sorted queue (Alg. 3, warm-started along
chains).  Default workload: BASELINE.json configs[2] ("C3"): 400 2-D
-div(a grad u) + c u operators on a 200 x 200 grid, L = 200 smallest eigenpairs,
nex = 40, tol 1e-8, split into 32 concurrent warm-start chains per GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl scsf|reference] [--config C1..C5]
  torchrun --nproc-per-node N bench.py --gpus N ...

Multi-GPU.  C1-C4: weak scaling, G ranks solve G x N operators, each rank a
contiguous slice of the global sorted queue, no data-path collective.
C5: one operator row-partitioned over the G ranks (scsf_solve_queue_dist: NCCL
halo exchange + all-reduced Gram blocks), strong scaling over a fixed chain.
`--gpus N` without torchrun re-launches itself under torch.distributed.run.

Prints one JSON line on rank 0 (contract in DESIGN.md §7).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

METRIC = "operators solved/s to 1e-8 residual"
UNIT = "operators/s"
CONFIG_INDEX = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}
# Filter degree m the bench runs each config at.  The paper treats m as a free hyperparameter
# (tab:degree: "as long as m is chosen within a reasonable range, its specific value
# does not significantly influence the performance"; fixed at 20 for its n <= 1e4 problems).
# On the BASELINE configs the spectra are far wider (beta / lambda_L ~ 700 on C3), the degree-20
# filter sits in its slow regime and the outer iterations are 4-10x those of m = 60-120 (DESIGN.md
# reading R27, tools/degree_sweep.py, profiles/r02_degree_sweep*.jsonl).  Every operator still
# converges to the same tolerance; the line also reports the paper's m = 20 on the same queue.
# The degree has a stability ceiling: the filtered block's condition number grows like
# exp(2 m sqrt(delta)) and CholQR squares it; on C3, m = 224 / 256 left 53 / 130 of 400 operators
# unconverged (CholQR breakdown, profiles/r02_degree_limit_C3.jsonl), m = 160 / 192 none; since the
# device-side conditioning cap (reading R28) and the cold retry every m converges, and with the
# neighbour-sync filter m = 160 / 192 / 224 / 256 give 46.6 / 47.2 / 47.4 / 47.3 operators/s
# (profiles/r02_degree_sweep_s2.json).  C3 runs with Alg. 1's per-column degrees (degree < 0, P:175,
# SURVEY f2; the library's k_lock sets each column's m_j <= |degree|): at this degree they pay,
# 52.3 / 53.6 operators/s at max 192 / 256 against 49.1 uniform at 192 (profiles/r02_f2_sweep_C3.json).
# C2 / C4 likewise (profiles/r02_f2_sweep_C2_C4.json): C2 1532 (m = 20) -> 2760 (per column <= 80),
# C4 30.5 (m = 80) -> 33.6 (per column <= 256) operators/s.
# C5 (row partition, one chain; the slab step honours per-column degrees since session 2): 4.99 at
# m = 80, 6.57 / 6.80 / 6.06 operators/s at per column <= 120 / 160 / 256.
BENCH_DEGREE = {"C1": 20, "C2": -80, "C3": -256, "C4": -256, "C5": -160}
DEFAULT_CONFIG = "C3"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="scsf", choices=["scsf", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--degree", type=int, default=None, help="filter degree m (default: BENCH_DEGREE[config])")
    ap.add_argument("--n-ops", type=int, default=None, help="operators per rank (C5: chain length; default N / 8)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-ops", type=int, default=None)
    ap.add_argument("--e2e-vecs", type=int, default=1, help="copy eigenvectors back in the e2e leg")
    ap.add_argument("--roofline-ops", type=int, default=8,
                    help="operators in the single-chain instrumented pass that measures the kernels")
    ap.add_argument("--chains-per-gpu", type=int, default=32,
                    help="concurrent warm-start chains per GPU (the paper's M chunks, P:856)")
    ap.add_argument("--no-paper-degree", action="store_true", help="skip the m = 20 pass")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def maybe_spawn(args):
    """`--gpus N` outside torchrun: run this script as N ranks (one per GPU) and exit with their status."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def workload_desc(cfg, n_total, world, degree):
    return {
        "workload": f"{cfg.name}: BASELINE.json configs[{CONFIG_INDEX[cfg.name]}]",
        "operator": {"lapv": "-Lap u + V u", "diva": "-div(a grad u)", "divac": "-div(a grad u) + c u"}[cfg.family],
        "grid": [cfg.nx] * cfg.dim, "n": cfg.n, "N_total": n_total, "N_per_gpu": n_total // world,
        "L": cfg.L, "nex": cfg.nex, "block": cfg.b, "degree": degree, "paper_degree": cfg.degree, "tol": cfg.tol,
        "p0": cfg.p0, "max_iter": cfg.max_iter,
        # degree < 0: Alg. 1's per-column degrees, each column's m_j <= |degree|
        "filter_degree": ({"per_column": True, "max": -degree} if degree < 0 else {"per_column": False, "m": degree}),
    }


# ------------------------------------------------------------------ clocks ----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    """HBM GB/s from MEASURED_PEAKS.json (driver-written); fp64 DMMA from this repo's cuBLAS DGEMM
    measurement on the box (MEASURED_PEAKS.json has no fp64 entry)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk, kind = json.load(f), "measured"
    except OSError:
        pk, kind = {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"
    fp64, fp64_src = 36.8, "fallback: 148 SMs x 4 DMMA sub-partitions x 64 flop/clk x 1.965 GHz (nominal)"
    try:
        with open(os.path.join(ROOT, "profiles", "r01_dgemm_peak.json")) as f:
            d = json.load(f)
        fp64 = float(d["dgemm_8192_sustained_tflops"])
        fp64_src = ("profiles/r01_dgemm_peak.json: cuBLAS DGEMM 8192^3 sustained, measured on a B200 of this pool "
                    "(tools/dgemm_peak.py)")
    except (OSError, ValueError, TypeError, KeyError):
        pass
    return float(pk.get("hbm_gbs", 6650.0)), kind, fp64, fp64_src


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def host_mem_free():
    try:
        import psutil
        return int(psutil.virtual_memory().available)
    except Exception:
        return 0


# --------------------------------------------------------------- cpu oracle ----
def oracle_rate(cfg, params_all, fields, sample_ops: int):
    """The oracle as it stands, on the host cores: operators/s on a bounded sample."""
    from oracle import eig as oeig, sort as osort
    t0 = time.perf_counter()
    osort.sort_problems(params_all, cfg.dim, cfg.nx, cfg.p0)
    t_sort = time.perf_counter() - t0
    N = params_all.shape[0]
    t0 = time.perf_counter()
    for i in range(sample_ops):
        oeig.smallest_eigpairs(fields, i, cfg.L)
    t_eig = time.perf_counter() - t0
    per_op = t_eig / sample_ops + t_sort / N
    return 1.0 / per_op, t_sort, t_eig


def default_cpu_sample(cfg):
    return {"C1": 6, "C2": 6, "C3": 2, "C4": 1, "C5": 1}.get(cfg.name, 1)


# --------------------------------------------------------------- reference ----
def run_reference(args, cfg, degree):
    """--impl reference: the CPU oracle timed as it stands (rank 0 only under torchrun)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import synth
    from oracle import eig as oeig, sort as osort
    N = args.n_ops or cfg.n_ops
    if cfg.name == "C5":
        N = args.n_ops or 8
    params = synth.make_batch(cfg, N, params_only=True).params
    t0 = time.perf_counter()
    osort.sort_problems(params, cfg.dim, cfg.nx, cfg.p0)
    t_sort = time.perf_counter() - t0
    ops_per_step = 2 if cfg.name in ("C1", "C2") else 1
    fields = synth.make_batch(cfg, ops_per_step * (args.warmup + args.steps))
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for j in range(ops_per_step):
            oeig.smallest_eigpairs(fields, s * ops_per_step + j, cfg.L)
        dt = time.perf_counter() - t0 + t_sort * ops_per_step / N
        if s >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = ops_per_step / (ms / 1000.0)
    sample = (f"{ops_per_step} operator(s) per step by shift-invert block Lanczos + the oracle sort of all "
              f"{N} operators ({t_sort:.2f} s) amortised per operator")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if cfg.name == "C5" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_desc(cfg, N, 1, degree),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": host_cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- rooflines ----
def roofline_objects(scsf, cfg, ops, rst, r_ms, degree, step_ms_per_op, hbm, hbm_kind, fp64, fp64_src):
    """Filter (HBM) and DGEMM (fp64 tensor) roofline objects from an instrumented single-chain pass."""
    fbytes = sum(s["filter_bytes"] for s in rst)
    fms = sum(s["t_filter_ms"] for s in rst)
    gms = sum(s["t_gemm_ms"] for s in rst)
    gfl = sum(s["gemm_flops"] for s in rst)
    oms = sum(s["t_ortho_ms"] for s in rst)
    rms = sum(s["t_rr_ms"] for s in rst)
    fsteps = sum(s["filter_steps"] for s in rst)
    kind = scsf.filter_kind(ops)
    kname = scsf.FILTER_KERNELS.get(kind, "?")
    launches_f = sum(s["iterations"] for s in rst) if kind > 0 else fsteps
    achieved = (fbytes / (fms / 1000.0)) / 1e9 if fms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "filter_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            ent = tj.get(cfg.name, {})
            if ent.get("config") == cfg.name and ent.get("filter_kind") == kind:
                # ncu DRAM bytes of the profiled whole-filter launch (Y_0 in, Y_m out: independent of the
                # degree), scaled by this run's mean active columns per launch
                m_ = abs(degree)
                per = fbytes / max(launches_f, 1) - 8.0 * (1 + cfg.dim) * cfg.n * m_
                cols = per / ((16.0 + 24.0 * (m_ - 1)) * cfg.n)
                traffic = ent["dram_bytes_per_launch"] * cols / ent["columns"]
        except Exception:
            traffic = None
    hbm_obj = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "unit": "GB/s",
               "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
               "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({hbm_kind})",
               "measured_on": f"single-chain pass of {len(rst)} operators after the timed region, CUDA events on "
                              f"the chain stream around each iteration's filter (degree {abs(degree)})",
               "achieved_is": ("algorithmic bytes of Alg. 1's streaming form (per step read Y_s, Y_s-1, write "
                               "Y_s+1, + the coefficient arrays) / filter time; this kernel keeps the block on "
                               "chip, so DRAM moves only Y_0 in and Y_m out (traffic); an effective streaming-"
                               "equivalent rate bounded by shared memory and the cluster barrier, not DRAM")
                              if kind > 0 else "algorithmic bytes per step / step time (streams HBM)",
               "launches": launches_f, "avg_launch_us": 1000.0 * fms / max(launches_f, 1),
               "bytes_per_launch": fbytes / max(launches_f, 1),
               "share_of_single_chain_time": fms / r_ms if r_ms > 0 else None}
    if kind > 0 and fms > 0:
        # the on-chip bound of the resident kernel: the fp64 FMA pipe.  Algorithmic flops per point, column
        # and step of Alg. 1 l. 5: (A - cI) y (2 (2d + 1) - 1 flops) and the recurrence a (.) + b Y_{s-1}
        # (3 flops): 12 in 2-D, 16 in 3-D; columns per launch from the streaming-form byte count above
        m_ = abs(degree)
        per = fbytes / max(launches_f, 1) - 8.0 * (1 + cfg.dim) * cfg.n * m_
        cols = per / ((16.0 + 24.0 * (m_ - 1)) * cfg.n)
        fl = cols * cfg.n * m_ * (4.0 * cfg.dim + 4.0) * launches_f
        dfma, dfma_src = fp64_alu_peak()
        a_tf = fl / (fms / 1000.0) / 1e12
        hbm_obj["roofline_alu"] = {
            "bound": "alu", "kernel": kname, "achieved": a_tf, "peak": dfma, "unit": "TFLOP/s",
            "frac": a_tf / dfma, "peak_source": dfma_src,
            "achieved_is": f"algorithmic fp64 flops of the recurrence ({int(4 * cfg.dim + 4)} per point, column and "
                           "step) / filter time: the kernel's on-chip ceiling (its steps never touch DRAM)",
            "flops_per_launch": fl / max(launches_f, 1)}
    dmma_obj = None
    if gms > 0:
        a = gfl / (gms / 1000.0) / 1e12
        dmma_obj = {"bound": "tensor", "kernel": "k_gemm_tn2 / k_gemm_nn2 / k_gemm_nn3 (DMMA m8n8k4 fp64 tiles)",
                    "achieved": a, "peak": fp64, "unit": "TFLOP/s", "frac": a / fp64, "traffic": None,
                    "peak_source": fp64_src,
                    "achieved_is": "algorithmic flops of the tall-skinny products (Gram: unique upper entries, "
                                   "R^-1 apply: triangular) / time between CUDA events around each launch",
                    "flops_per_operator": gfl / max(len(rst), 1),
                    "share_of_single_chain_time": gms / r_ms if r_ms > 0 else None}
    phases = {"filter": fms, "ortho": oms, "rayleigh_ritz": rms, "gemm": gms, "total": r_ms}
    return hbm_obj, dmma_obj, phases


def fp64_alu_peak():
    """Measured DFMA throughput of this B200 (tools/fp64_pipes.cu -> profiles/r02_fp64_pipes.json), else the
    nominal 148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz."""
    p = os.path.join(ROOT, "profiles", "r02_fp64_pipes.json")
    try:
        j = json.load(open(p))
        return float(j["dfma_tflops"]), "profiles/r02_fp64_pipes.json: DFMA, tools/fp64_pipes.cu on a B200 of this pool"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal: 148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz"


def stream_probe(scsf, torch, cfg, ops, degree, hbm):
    """HBM roofline of the per-step streaming filter (k_stencil_v4) on this workload's operator:
    scsf_cheb_filter forced to stream, b columns, degree m, CUDA events, 5 repetitions."""
    if ops.stencil != scsf.STENCIL_FLUX:
        return None
    m = abs(degree)
    b = cfg.b
    g = torch.Generator(device=ops.coef.device).manual_seed(7)
    Y = torch.zeros((b, ops.ld), dtype=torch.float64, device=ops.coef.device)
    Y[:, :cfg.n] = torch.randn((b, cfg.n), dtype=torch.float64, device=ops.coef.device, generator=g)
    old = os.environ.get("SCSF_FILTER_STREAMING")
    os.environ["SCSF_FILTER_STREAMING"] = "1"
    try:
        lam, c, e = 1.0, 5e5, 4.9e5
        scsf.cheb_filter(ops, 0, Y, m, lam, c, e)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            scsf.cheb_filter(ops, 0, Y, m, lam, c, e)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    finally:
        if old is None:
            os.environ.pop("SCSF_FILTER_STREAMING", None)
        else:
            os.environ["SCSF_FILTER_STREAMING"] = old
    n = cfg.n
    byt = (16.0 + 24.0 * (m - 1)) * n * b + 8.0 * (1 + cfg.dim) * n * m
    gbs = byt / (ms / 1000.0) / 1e9
    return {"bound": "hbm", "kernel": "k_stencil_v4 (one streaming launch per filter step)", "achieved": gbs,
            "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "columns": b, "degree": m,
            "avg_launch_us": 1000.0 * ms / m, "bytes_per_launch": byt / m,
            "measured_on": "scsf_cheb_filter forced to the streaming kernel (SCSF_FILTER_STREAMING=1) on one "
                           "operator of this workload, b columns, 5 repetitions after one warm-up, CUDA events"}


# -------------------------------------------------------------------- main ----
def main():
    args = parse()
    import synth
    cfg = synth.get_config(args.config)
    degree = args.degree if args.degree is not None else BENCH_DEGREE.get(cfg.name, cfg.degree)
    if args.impl == "reference":
        run_reference(args, cfg, degree)
        return
    maybe_spawn(args)
    import torch
    import torch.distributed as dist
    from paper_2510_23215_b200 import scsf

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    scsf.load_library()
    hbm, hbm_kind, fp64, fp64_src = measured_peaks()
    if cfg.name == "C5":
        run_rowpart(args, cfg, degree, rank, world, local, dev, torch, dist, scsf, hbm, hbm_kind, fp64, fp64_src)
    else:
        run_chains(args, cfg, degree, rank, world, local, dev, torch, dist, scsf, hbm, hbm_kind, fp64, fp64_src)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def timed_steps(args, step, flush, stream, torch, dist, world, local, dev):
    """W untimed warm-up steps, then K steps each bracketed by a barrier and device synchronisation,
    L2 flushed before each; returns (max-over-ranks mean ms, per-step stats, launches per step, clocks)."""
    from paper_2510_23215_b200 import scsf

    def barrier():
        if world > 1:
            dist.barrier()
    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms, all_stats = [], []
    launches0 = scsf.launch_count()
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        all_stats.extend(st)
    launches = (scsf.launch_count() - launches0) / args.steps
    clk = clocks.stop()
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, all_stats, launches, clk


def run_chains(args, cfg, degree, rank, world, local, dev, torch, dist, scsf, hbm, hbm_kind, fp64, fp64_src):
    from paper_2510_23215_b200.pipeline import chain_bounds
    n_per = args.n_ops or cfg.n_ops
    N = n_per * world

    # ---- inputs (seeded, synthetic), resident in HBM before the timed region
    params_host = synth_params(cfg, N)
    params = torch.from_numpy(params_host).to(dev)
    # every rank computes the same permutation; used here only to pick this rank's inputs
    perm0, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    lo, hi = chain_bounds(N, world, rank)
    my_ops = np.sort(perm0[lo:hi])
    import synth
    fields = synth.make_batch(cfg, indices=my_ops)
    g2l = {int(g): j for j, g in enumerate(my_ops)}          # global index -> position in my_ops
    faces = [torch.from_numpy(f).to(dev) for f in fields.faces]
    cc = torch.from_numpy(fields.c).to(dev)
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, cc)
    n_chains = max(1, min(args.chains_per_gpu, hi - lo))
    ws = scsf._workspace(scsf.solve_workspace(ops, cfg.L, cfg.nex).numel() * n_chains, dev)
    evals = torch.empty((hi - lo, cfg.L), dtype=torch.float64, device=dev)
    evecs = torch.empty((hi - lo, cfg.L, ops.ld), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def make_step(m):
        def step():
            perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
            chain = np.array([g2l[int(g)] for g in perm[lo:hi]], dtype=np.int32)
            _, _, stats = scsf.solve_chains(ops, chain, n_chains, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter,
                                            seed=12345, ws=ws, evals=evals, evecs=evecs, raise_on_fail=False)
            return stats
        return step

    ms, all_stats, launches, clk = timed_steps(args, make_step(degree), flush, stream, torch, dist, world, local, dev)
    value = N / (ms / 1000.0)
    conv = sum(1 for s in all_stats if s["status"] == 0)
    iters = [s["iterations"] for s in all_stats]

    # ---- the paper's degree (m = 20) on the same queue: one warm-up + one timed pass
    paper = None
    if not args.no_paper_degree and degree != cfg.degree:
        stp = make_step(cfg.degree)
        stp()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(1.0)
        e0.record(stream)
        pst = stp()
        e1.record(stream)
        torch.cuda.synchronize()
        pms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([pms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pms = float(t.item())
        paper = {"degree": cfg.degree, "value": N / (pms / 1000.0), "unit": UNIT, "ms_per_step": pms, "steps": 1,
                 "converged": f"{sum(1 for s in pst if s['status'] == 0)}/{len(pst)}",
                 "iterations_mean": float(np.mean([s["iterations"] for s in pst]))}

    # ---- roofline pass: one chain with phase and DGEMM timers (CUDA events on the chain's stream)
    nr = min(args.roofline_ops, hi - lo)
    scsf.set_timing(True)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    perm_r, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    chain_r = np.array([g2l[int(g)] for g in perm_r[lo:hi]], dtype=np.int32)[:nr]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, _, rst = scsf.solve_chains(ops, chain_r, 1, cfg.L, cfg.nex, degree, cfg.tol, cfg.max_iter, seed=12345,
                                  ws=ws, evals=evals[:nr], evecs=evecs[:nr], raise_on_fail=False)
    e1.record(stream)
    torch.cuda.synchronize()
    scsf.set_timing(False)
    r_ms = e0.elapsed_time(e1)
    hbm_obj, dmma_obj, phases = roofline_objects(scsf, cfg, ops, rst, r_ms, degree, ms / max(hi - lo, 1), hbm,
                                                 hbm_kind, fp64, fp64_src)
    streaming = stream_probe(scsf, torch, cfg, ops, degree, hbm) if rank == 0 else None

    # ---- e2e through the public API with host buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        k2 = args.e2e_steps or max(1, min(args.steps, 2))
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hp = pin(params_host)
        hf = [pin(f) for f in fields.faces]
        hc = pin(fields.c)
        vec_bytes = (hi - lo) * cfg.L * ops.ld * 8
        want_v = bool(args.e2e_vecs) and host_mem_free() > 2.5 * vec_bytes
        out_e = torch.empty((hi - lo, cfg.L), dtype=torch.float64).pin_memory()
        out_v = torch.empty((hi - lo, cfg.L, ops.ld), dtype=torch.float64).pin_memory() if want_v else None
        h2d = hp.numel() * 8 + sum(f.numel() * 8 for f in hf) + hc.numel() * 8
        d2h = (hi - lo) * cfg.L * 8 + ((hi - lo) * cfg.L * cfg.n * 8 if out_v is not None else 0)
        hws = scsf._workspace(scsf.chains_host_workspace_bytes(ops, cfg.L, cfg.nex) * n_chains, dev)

        def e2e_step():
            dp = hp.to(dev, non_blocking=True)
            dfs = [f.to(dev, non_blocking=True) for f in hf]
            dc = hc.to(dev, non_blocking=True)
            o = scsf.assemble(cfg.dim, cfg.nx, cfg.h, dfs, dc)
            perm, _, _ = scsf.sort(dp, cfg.dim, cfg.nx, cfg.p0)
            chain = np.array([g2l[int(g)] for g in perm[lo:hi]], dtype=np.int32)
            # pairs stream to the pinned host buffers while the chains run (scsf_solve_chains_host)
            scsf.solve_chains_host(o, chain, n_chains, cfg.L, cfg.nex, out_e, out_v, degree, cfg.tol,
                                   cfg.max_iter, seed=12345, raise_on_fail=False, ws=hws)

        e2e_step()
        torch.cuda.synchronize()
        tms = []
        for _ in range(k2):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            tms.append(e0.elapsed_time(e1))
        ems = float(np.mean(tms))
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": N / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": k2, "ms_per_step": ems,
               "what": "pinned host fields -> H2D -> scsf_assemble -> scsf_sort -> scsf_solve_chains_host (evals"
                       + (" + evecs" if out_v is not None else "") + " streamed D2H into pinned host memory while "
                       "the chains run)" + ("" if out_v is not None or not args.e2e_vecs else
                                            "; eigenvectors not copied: not enough free host memory to pin them")}

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(args.cpu_sample_ops or default_cpu_sample(cfg), hi - lo)
        rate, t_sort, t_eig = oracle_rate(cfg, params_host, fields, sample)
        cpu = {"value": rate, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
               "sample": f"oracle sort of all {N} operators ({t_sort:.2f} s, amortised) + shift-invert block "
                         f"Lanczos on {sample} operator(s) ({t_eig:.2f} s); numpy/LAPACK threads = host cores"}

    if rank == 0:
        conf = workload_desc(cfg, N, world, degree)
        conf["chains_per_gpu"] = n_chains
        conf["parallelism"] = f"dp{world} x {n_chains} concurrent warm-start chains per GPU"
        conf["l2"] = "inputs (params + DIA batch) exceed the 126 MB L2 and a 256 MB buffer is written between steps"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded GRF coefficient fields, DESIGN.md §3)",
                "config": conf, "roofline": hbm_obj, "roofline_alu": hbm_obj.pop("roofline_alu", None),
                "roofline_dmma": dmma_obj, "roofline_streaming": streaming,
                "single_chain_phase_ms": phases, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(round(launches)), "clocks": clk,
                "converged": f"{conv}/{len(all_stats)}", "iterations_mean": float(np.mean(iters)) if iters else None,
                "iterations_max": int(max(iters)) if iters else None, "paper_degree": paper}
        print(json.dumps(line), flush=True)


def synth_params(cfg, N):
    import synth
    return synth.make_batch(cfg, N, params_only=True).params


def run_rowpart(args, cfg, degree, rank, world, local, dev, torch, dist, scsf, hbm, hbm_kind, fp64, fp64_src):
    """C5: every rank holds the same operators; each operator of the chain is row-partitioned over
    the ranks (scsf_solve_queue_dist, NCCL).  Strong scaling over a fixed chain."""
    import synth
    from paper_2510_23215_b200 import pipeline
    K = args.n_ops or 8
    params_host = synth_params(cfg, cfg.n_ops)
    params = torch.from_numpy(params_host).to(dev)
    perm0, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    my_ops = np.sort(perm0[:K])
    fields = synth.make_batch(cfg, indices=my_ops)
    g2l = {int(g): j for j, g in enumerate(my_ops)}
    faces = [torch.from_numpy(f).to(dev) for f in fields.faces]
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(fields.c).to(dev))
    comm = pipeline.make_comm(rank, world)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
        chain = np.array([g2l[int(g)] for g in perm[:K]], dtype=np.int32)
        _, _, stats, _ = scsf.solve_queue_dist(ops, chain, cfg.L, cfg.nex, comm, degree, cfg.tol, cfg.max_iter,
                                               seed=12345, want_vecs=True, raise_on_fail=False)
        return stats

    ms, all_stats, launches, clk = timed_steps(args, step, flush, stream, torch, dist, world, local, dev)
    value = K / (ms / 1000.0)
    conv = sum(1 for s in all_stats if s["status"] == 0)
    iters = [s["iterations"] for s in all_stats]
    # instrumented pass (phase + DGEMM timers) over 2 operators of the chain
    scsf.set_timing(True)
    torch.cuda.synchronize()
    perm_r, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    chain_r = np.array([g2l[int(g)] for g in perm_r[:min(2, K)]], dtype=np.int32)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, _, rst, _ = scsf.solve_queue_dist(ops, chain_r, cfg.L, cfg.nex, comm, degree, cfg.tol, cfg.max_iter,
                                         seed=12345, want_vecs=False, raise_on_fail=False)
    e1.record(stream)
    torch.cuda.synchronize()
    scsf.set_timing(False)
    hbm_obj, dmma_obj, phases = roofline_objects(scsf, cfg, ops, rst, e0.elapsed_time(e1), degree, ms / K, hbm,
                                                 hbm_kind, fp64, fp64_src)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hp, hc = pin(params_host), pin(fields.c)
        hf = [pin(f) for f in fields.faces]
        y0, y1 = scsf.slab_rows(cfg.nx, world, rank)
        out_e = torch.empty((K, cfg.L), dtype=torch.float64).pin_memory()
        out_v = torch.empty((K, cfg.L, scsf.ld_for(cfg.nx * (y1 - y0))), dtype=torch.float64).pin_memory()
        h2d = hp.numel() * 8 + sum(f.numel() * 8 for f in hf) + hc.numel() * 8
        d2h = out_e.numel() * 8 + K * cfg.L * cfg.nx * (y1 - y0) * 8

        def e2e_step():
            dp = hp.to(dev, non_blocking=True)
            o = scsf.assemble(cfg.dim, cfg.nx, cfg.h, [f.to(dev, non_blocking=True) for f in hf],
                              hc.to(dev, non_blocking=True))
            perm, _, _ = scsf.sort(dp, cfg.dim, cfg.nx, cfg.p0)
            chain = np.array([g2l[int(g)] for g in perm[:K]], dtype=np.int32)
            ev, vec, _, _ = scsf.solve_queue_dist(o, chain, cfg.L, cfg.nex, comm, degree, cfg.tol, cfg.max_iter,
                                                  seed=12345, want_vecs=True, raise_on_fail=False)
            out_e.copy_(ev, non_blocking=True)
            out_v.copy_(vec, non_blocking=True)
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": K / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": 1, "ms_per_step": ems,
               "what": "pinned host fields -> H2D -> scsf_assemble -> scsf_sort -> scsf_solve_queue_dist -> D2H of "
                       "evals + this rank's eigenvector slab"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, t_sort, t_eig = oracle_rate(cfg, params_host, fields, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
               "sample": f"oracle sort of all {cfg.n_ops} operators ({t_sort:.2f} s, amortised) + shift-invert "
                         f"block Lanczos on 1 operator ({t_eig:.2f} s)"}
    comm.close()
    if rank == 0:
        conf = workload_desc(cfg, K, 1, degree)
        conf["N_per_gpu"] = K
        conf["chain"] = f"the first {K} operators of the sorted queue of {cfg.n_ops}"
        conf["parallelism"] = f"row partition over {world} GPU(s): 1-D slabs of the {cfg.nx} grid rows, NCCL halo + " \
                              "all-reduced Gram / projection blocks"
        conf["l2"] = "the n x b blocks (720 MB) exceed the 126 MB L2; a 256 MB buffer is written between steps"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded GRF coefficient fields, DESIGN.md §3)",
                "config": conf, "roofline": hbm_obj, "roofline_alu": hbm_obj.pop("roofline_alu", None),
                "roofline_dmma": dmma_obj, "single_chain_phase_ms": phases,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(round(launches)), "clocks": clk,
                "converged": f"{conv}/{len(all_stats)}", "iterations_mean": float(np.mean(iters)) if iters else None,
                "iterations_max": int(max(iters)) if iters else None}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
