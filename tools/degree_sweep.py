"""Filter degree m / extra columns nex sweep (SURVEY §8(d) tuning; paper tab:degree P:1026-1040).

For each config, degree and nex: one untimed pass (fills the CUDA-graph cache), then one timed
pass over a seeded prefix of the sorted queue in C concurrent chains.  Reports operators/s,
mean / max outer iterations and SpMM columns per operator.  Results do not depend on m or nex
(every operator converges to the same tolerance); the cost does.

  python tools/degree_sweep.py C3:64:32 C4:64:32 --m 20,30,40,60 --nex 0    (nex 0 = config default)
"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+", help="CFG:N:CHAINS")
    ap.add_argument("--m", default="20,30,40")
    ap.add_argument("--nex", default="0")
    ap.add_argument("--max-iter", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    for spec in a.specs:
        name, N, C = spec.split(":")
        N, C = int(N), int(C)
        cfg = synth.get_config(name)
        f = synth.make_batch(cfg, N)
        params = torch.from_numpy(f.params).to(dev)
        if f.is_vib:
            ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
        else:
            faces = [torch.from_numpy(x).to(dev) for x in f.faces]
            ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
        perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
        for nex in [int(x) for x in a.nex.split(",")]:
            nex = nex or cfg.nex
            ws = scsf._workspace(scsf.solve_workspace(ops, cfg.L, nex).numel() * C, dev)
            for m in [int(x) for x in a.m.split(",")]:
                mi = a.max_iter or cfg.max_iter
                kw = dict(seed=3, want_vecs=False, raise_on_fail=False, ws=ws)
                scsf.solve_chains(ops, perm, C, cfg.L, nex, m, cfg.tol, mi, **kw)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _, _, st = scsf.solve_chains(ops, perm, C, cfg.L, nex, m, cfg.tol, mi, **kw)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                its = np.array([s["iterations"] for s in st], dtype=float)
                cols = np.array([s["spmm_columns"] for s in st], dtype=float)
                warm = np.array([s["warm"] for s in st], dtype=bool)
                row = {"config": name, "N": N, "chains": C, "m": m, "nex": nex, "b": cfg.L + nex,
                       "operators_per_s": N / (ms / 1e3), "ms": ms,
                       "converged": int(sum(s["status"] == 0 for s in st)),
                       "iterations_mean": float(its.mean()), "iterations_max": int(its.max()),
                       "iterations_warm_mean": float(its[warm].mean()) if warm.any() else None,
                       "iterations_cold_mean": float(its[~warm].mean()) if (~warm).any() else None,
                       "spmm_columns_mean": float(cols.mean())}
                print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
