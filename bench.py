#!/usr/bin/env python
"""bench.py — SCSF hot path on B200: truncated-FFT sort + warm-started ChFSI.

One step = one pass of the whole hot path over this rank's share of the
workload: scsf_sort over the global queue (every rank computes the same
permutation) + scsf_solve_queue over the rank's contiguous chain.  The
workload (config.workload) is BASELINE.json configs[1] ("C2"): 1000 2-D
-Lap u + V u operators on a 100x100 grid, L = 100 smallest eigenpairs,
nex = 20, degree 20, tol 1e-8.  Weak scaling: with G ranks the global queue
holds G x 1000 operators (operator i is a pure function of its index).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl scsf|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints one JSON line on rank 0 (contract in DESIGN.md §7).
"""
from __future__ import annotations

import argparse
import json
import math
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="scsf", choices=["scsf", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n-ops", type=int, default=None, help="operators per rank (default: the config's N)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-ops", type=int, default=6)
    ap.add_argument("--e2e-vecs", type=int, default=1, help="copy eigenvectors back in the e2e leg")
    ap.add_argument("--roofline-ops", type=int, default=64,
                    help="operators in the single-chain instrumented pass that measures the filter kernel")
    ap.add_argument("--chains-per-gpu", type=int, default=32,
                    help="concurrent warm-start chains per GPU (the paper's M chunks, P:856)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg, n_total, world):
    return {
        "workload": f"{cfg.name}: BASELINE.json configs[{['C1','C2','C3','C4','C5'].index(cfg.name)}]",
        "operator": {"lapv": "-Lap u + V u", "diva": "-div(a grad u)", "divac": "-div(a grad u) + c u"}[cfg.family],
        "grid": [cfg.nx] * cfg.dim, "n": cfg.n, "N_total": n_total, "N_per_gpu": n_total // world,
        "L": cfg.L, "nex": cfg.nex, "block": cfg.b, "degree": cfg.degree, "tol": cfg.tol, "p0": cfg.p0,
        "chains": world, "parallelism": f"chains{world}",
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
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def lib_ws_host(ops, cfg):
    import ctypes
    from paper_2510_23215_b200 import scsf
    st = ops.c_struct()
    return scsf.load_library().scsf_solve_chains_host_workspace_bytes(ctypes.byref(st), cfg.L, cfg.nex)


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


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


# --------------------------------------------------------------- reference ----
def run_reference(args, cfg):
    """--impl reference: the CPU oracle timed as it stands (rank 0 only under torchrun)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import synth
    from oracle import eig as oeig, sort as osort
    N = args.n_ops or cfg.n_ops
    params = synth.make_batch(cfg, N, params_only=True).params
    t0 = time.perf_counter()
    osort.sort_problems(params, cfg.dim, cfg.nx, cfg.p0)
    t_sort = time.perf_counter() - t0
    ops_per_step = 2
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
    sample = (f"{ops_per_step} operators per step by shift-invert block Lanczos + the oracle sort of all "
              f"{N} operators ({t_sort:.2f} s) amortised per operator")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(cfg, N, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": host_cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- main ----
def main():
    args = parse()
    import synth
    cfg = synth.get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import torch.distributed as dist
    from paper_2510_23215_b200 import scsf
    from paper_2510_23215_b200.pipeline import chain_bounds

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    scsf.load_library()
    n_per = args.n_ops or cfg.n_ops
    N = n_per * world

    # ---- inputs (seeded, synthetic), resident in HBM before the timed region
    params_host = synth.make_batch(cfg, N, params_only=True).params
    params = torch.from_numpy(params_host).to(dev)
    # every rank computes the same permutation; used here only to pick this rank's inputs
    perm0, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    lo, hi = chain_bounds(N, world, rank)
    my_ops = np.sort(perm0[lo:hi])
    fields = synth.make_batch(cfg, indices=my_ops)
    # local operator numbering: global index -> position in my_ops
    g2l = {int(g): j for j, g in enumerate(my_ops)}
    faces = [torch.from_numpy(f).to(dev) for f in fields.faces]
    cc = torch.from_numpy(fields.c).to(dev)
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, cc)
    n_chains = max(1, min(args.chains_per_gpu, hi - lo))
    ws = scsf._workspace(scsf.solve_workspace(ops, cfg.L, cfg.nex).numel() * n_chains, dev)
    evals = torch.empty((hi - lo, cfg.L), dtype=torch.float64, device=dev)
    evecs = torch.empty((hi - lo, cfg.L, ops.ld), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
        chain = np.array([g2l[int(g)] for g in perm[lo:hi]], dtype=np.int32)
        _, _, stats = scsf.solve_chains(ops, chain, n_chains, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter,
                                        seed=12345, ws=ws, evals=evals, evecs=evecs, raise_on_fail=False)
        return stats

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (phase timers off)
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
    ms_local = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    else:
        ms = ms_local
    value = N / (ms / 1000.0)

    conv = sum(1 for s in all_stats if s["status"] == 0)
    iters = [s["iterations"] for s in all_stats]

    # ---- roofline pass: the dominant kernel (filter step) timed live with CUDA events on the
    # launching stream, one chain (concurrent chains would overlap each other's phases)
    nr = min(args.roofline_ops, hi - lo)
    scsf.set_timing(True)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    perm_r, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    chain_r = np.array([g2l[int(g)] for g in perm_r[lo:hi]], dtype=np.int32)[:nr]
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, _, rst = scsf.solve_chains(ops, chain_r, 1, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=12345,
                                  ws=ws, evals=evals[:nr], evecs=evecs[:nr], raise_on_fail=False)
    e1.record(stream)
    torch.cuda.synchronize()
    scsf.set_timing(False)
    r_ms = e0.elapsed_time(e1)
    fbytes = sum(s["filter_bytes"] for s in rst)
    fms = sum(s["t_filter_ms"] for s in rst)
    oms = sum(s["t_ortho_ms"] for s in rst)
    rms = sum(s["t_rr_ms"] for s in rst)
    fsteps = sum(s["filter_steps"] for s in rst)
    peaks, peak_kind = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = (fbytes / (fms / 1000.0)) / 1e9 if fms > 0 else None
    kind = scsf.filter_kind(ops)
    kname = scsf.FILTER_KERNELS.get(kind, "?")
    # one launch = a whole filter (m steps) for the resident kernels, one step for the streaming one
    launches_f = sum(s["iterations"] for s in rst) if kind > 0 else fsteps
    traffic = None
    tp = os.path.join(ROOT, "profiles", "filter_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("config") == cfg.name and tj.get("filter_kind") == kind:
                # ncu DRAM bytes of the profiled launch, scaled by this run's mean launch size
                traffic = tj["dram_bytes_per_launch"] * (fbytes / max(launches_f, 1)) / tj["algorithmic_bytes_per_launch"]
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved,
                "peak": hbm, "unit": "GB/s", "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "measured_on": f"single-chain pass of {nr} operators after the timed region, CUDA events on the "
                               f"chain stream around each iteration's filter ({cfg.degree} steps)",
                "achieved_is": ("algorithmic bytes of Alg. 1's streaming form (read Y_s, Y_s-1, write Y_s+1 per "
                                "step) / filter time; the resident kernels keep the block on chip, so HBM moves "
                                "only Y_0 in and Y_m out (see traffic)") if kind > 0 else
                               "algorithmic bytes per step / step time",
                "launches": launches_f, "avg_launch_us": 1000.0 * fms / max(launches_f, 1),
                "bytes_per_launch": fbytes / max(launches_f, 1),
                "share_of_single_chain_step": fms / r_ms if r_ms > 0 else None,
                "single_chain_phase_ms": {"filter": fms, "ortho": oms, "rayleigh_ritz": rms, "total": r_ms}}

    # ---- e2e through the public API with host buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        from paper_2510_23215_b200 import pipeline
        k2 = args.e2e_steps or max(1, min(args.steps, 2))
        host_faces = [np.ascontiguousarray(f) for f in fields.faces]
        pin = lambda a: torch.from_numpy(a).pin_memory()
        hp = pin(params_host)
        hf = [pin(f) for f in host_faces]
        hc = pin(fields.c)
        out_e = torch.empty((hi - lo, cfg.L), dtype=torch.float64).pin_memory()
        out_v = torch.empty((hi - lo, cfg.L, ops.ld), dtype=torch.float64).pin_memory() if args.e2e_vecs else None
        h2d = hp.numel() * 8 + sum(f.numel() * 8 for f in hf) + hc.numel() * 8
        d2h = (hi - lo) * cfg.L * 8 + ((hi - lo) * cfg.L * cfg.n * 8 if out_v is not None else 0)

        hws = scsf._workspace(lib_ws_host(ops, cfg) * n_chains, dev)

        def e2e_step():
            dp = hp.to(dev, non_blocking=True)
            dfs = [f.to(dev, non_blocking=True) for f in hf]
            dc = hc.to(dev, non_blocking=True)
            o = scsf.assemble(cfg.dim, cfg.nx, cfg.h, dfs, dc)
            perm, _, _ = scsf.sort(dp, cfg.dim, cfg.nx, cfg.p0)
            chain = np.array([g2l[int(g)] for g in perm[lo:hi]], dtype=np.int32)
            # pairs stream to the pinned host buffers while the chains run (scsf_solve_chains_host)
            scsf.solve_chains_host(o, chain, n_chains, cfg.L, cfg.nex, out_e, out_v, cfg.degree, cfg.tol,
                                   cfg.max_iter, seed=12345, raise_on_fail=False, ws=hws)

        e2e_step()
        torch.cuda.synchronize()
        tms = []
        for _ in range(k2):
            barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
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
                       "the chains run)"}

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(args.cpu_sample_ops, hi - lo)
        rate, t_sort, t_eig = oracle_rate(cfg, params_host, fields, sample)
        cpu = {"value": rate, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
               "sample": f"oracle sort of all {N} operators ({t_sort:.2f} s, amortised) + shift-invert block "
                         f"Lanczos on {sample} operators ({t_eig:.2f} s); numpy/LAPACK threads = host cores"}

    if rank == 0:
        conf = workload_desc(cfg, N, world)
        conf["chains_per_gpu"] = n_chains
        conf["parallelism"] = f"dp{world} x {n_chains} concurrent chains per GPU"
        conf["l2"] = "inputs (params + DIA batch) exceed the 126 MB L2 and a 256 MB buffer is written between steps"
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded GRF coefficient fields, DESIGN.md §3)",
                "config": conf, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(round(launches)), "clocks": clk,
                "converged": f"{conv}/{len(all_stats)}", "iterations_mean": float(np.mean(iters)) if iters else None,
                "iterations_max": int(max(iters)) if iters else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
