"""the paper's similarity experiment on B200 (tab:perturbation_impact).

Batches of N perturbations of one base C2 operator (-Lap u + V u, 100 x 100, L = 100; the paper's
Helmholtz stand-in; synth.make_perturbed: V_i = V_base exp(size g_i), size = RMS relative
perturbation), plus the standard C2 generation.  Per batch and mode, one chain on one GPU:
  scsf      truncated-FFT sorted queue, warm start along the chain (the method)
  no-sort   warm start along the generation order (SCSF w/o sort)
  chfsi     every operator from a seeded random block (plain ChFSI; the paper's "independent")
Reports mean outer iterations and ms per operator.  Iteration counts are hardware-independent.

  python tools/similarity_sweep.py [N] [degree]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def solve(ops, cfg, chain, m, cold_each):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cold_each:
        st = [scsf.solve_one(ops, int(i), cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=77,
                             raise_on_fail=False)[2] for i in chain]
    else:
        _, _, st = scsf.solve_queue(ops, chain, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=77,
                                    want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = np.array([s["iterations"] for s in st], dtype=float)
    return {"iterations_mean": float(its.mean()), "iterations_max": int(its.max()),
            "converged": int(sum(s["status"] == 0 for s in st)), "ms_per_operator": 1e3 * dt / len(chain)}


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = synth.get_config("C2")
    dev = torch.device("cuda", 0)
    batches = [(f"perturbation {int(100 * s) if s >= 0.01 else s * 100:g}%", synth.make_perturbed(cfg, N, s))
               for s in (0.5, 0.1, 0.01, 0.0)]
    batches.append(("standard generation", synth.make_batch(cfg, N)))
    out = {"config": "C2 grid, L = 100, tol 1e-8", "N": N, "degree": m, "rows": []}
    warm = True
    for name, f in batches:
        faces = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in f.faces]
        ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(np.ascontiguousarray(f.c)).to(dev))
        params = torch.from_numpy(np.ascontiguousarray(f.params)).to(dev)
        perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
        if warm:                                            # CUDA-graph cache / first-launch costs
            solve(ops, cfg, perm[:4], m, False)
            warm = False
        row = {"batch": name,
               "scsf": solve(ops, cfg, perm, m, False),
               "no-sort": solve(ops, cfg, np.arange(N, dtype=np.int32), m, False),
               "chfsi": solve(ops, cfg, np.arange(N, dtype=np.int32), m, True)}
        print(json.dumps(row), file=sys.stderr, flush=True)
        out["rows"].append(row)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
