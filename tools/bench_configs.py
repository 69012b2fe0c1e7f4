"""Operators/s on every BASELINE.json config (one B200), the bench.py way: inputs resident,
sorted queue, C concurrent chains, CUDA events around the solve.  Full N for C1/C2; a seeded
prefix of the batch for C3/C4/C5 (their per-operator cost makes a full pass minutes long).
One untimed pass first (it fills the CUDA-graph cache, as bench.py's warm-up steps do).
Prints one JSON object.   python tools/bench_configs.py
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402

# (operators, chains).  C1 has only 64 operators: 16 chains of 4 keep every chain warm-started
# after its head (8 chains: ~1190, 16: ~1800, 32: ~2430 operators/s with half the solves cold).
PLAN = {"C1": (64, 16), "C2": (1000, 32), "C3": (64, 32), "C4": (64, 32), "C5": (8, 8), "V1": (200, 32)}


def main():
    names = sys.argv[1:] or list(PLAN)
    out = {}
    dev = torch.device("cuda", 0)
    for name in names:
        cfg = synth.get_config(name)
        N, C = PLAN[name]
        f = synth.make_batch(cfg, N)
        params = torch.from_numpy(f.params).to(dev)
        if f.is_vib:
            ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
        else:
            faces = [torch.from_numpy(x).to(dev) for x in f.faces]
            ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
        perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
        ws = scsf._workspace(scsf.solve_workspace(ops, cfg.L, cfg.nex).numel() * C, dev)   # reused, as bench.py
        scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter,
                          seed=3, want_vecs=False, raise_on_fail=False, ws=ws)    # warm-up pass (graph cache)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, _, st = scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=3,
                                     want_vecs=False, raise_on_fail=False, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        its = [s["iterations"] for s in st]
        out[name] = {"operators": N, "chains": C, "n": cfg.n, "L": cfg.L, "b": cfg.b,
                     "filter_kernel": ("k_stencil_vib (13-point streaming launch per filter step, Alg. 1)"
                                       if ops.stencil == scsf.STENCIL_VIB13 else
                                       scsf.FILTER_KERNELS[scsf.filter_kind(ops)]),
                     "operators_per_s": N / (ms / 1e3), "ms": ms,
                     "converged": int(sum(s["status"] == 0 for s in st)),
                     "iterations_mean": float(np.mean(its)), "iterations_max": int(max(its))}
        print(name, json.dumps(out[name]), flush=True, file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
