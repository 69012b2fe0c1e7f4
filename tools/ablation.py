"""the paper's method ablation on B200 (tab:sort1 / tab:sort3).

Modes over the same N operators (iteration counts are hardware-independent; time is this GPU):
  scsf        sorted queue (truncated-FFT greedy, p0 = 20), warm start along the chain
  full-sort   greedy on the raw fields (p0 = p, the SKR baseline of tab:sort2)
  no-sort     warm start along the original index order
  random      every operator from a seeded random block (plain ChFSI)
One chain (single-chain latency) per mode.  Writes one JSON object to stdout.

  python tools/ablation.py [CFG] [N] [DEGREE]
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def run(ops, cfg, chain, cold_each, m):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if cold_each:
        st = []
        for i in chain:
            _, _, s = scsf.solve_one(ops, int(i), cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=77,
                                     raise_on_fail=False)
            st.append(s)
    else:
        _, _, st = scsf.solve_queue(ops, chain, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=77,
                                    want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = np.array([s["iterations"] for s in st], dtype=float)
    cols = np.array([s["spmm_columns"] for s in st], dtype=float)
    return {"operators": len(chain), "converged": int(sum(s["status"] == 0 for s in st)),
            "iterations_mean": float(its.mean()), "iterations_max": int(its.max()),
            "spmm_columns_mean": float(cols.mean()), "ms_per_operator": 1e3 * dt / len(chain)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    cfg = synth.get_config(name)
    m = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.degree
    f = synth.make_batch(cfg, N)
    dev = torch.device("cuda", 0)
    params = torch.from_numpy(f.params).to(dev)
    if f.is_vib:
        ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
    else:
        faces = [torch.from_numpy(x).to(dev) for x in f.faces]
        ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
    perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    perm_full, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.nx)
    scsf.solve_queue(ops, perm[:2], cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, want_vecs=False)  # warm-up
    out = {"config": name, "N": N, "degree": m, "tol": cfg.tol, "L": cfg.L, "nex": cfg.nex,
           "scsf": run(ops, cfg, perm, False, m),
           "full-sort": run(ops, cfg, perm_full, False, m),
           "no-sort": run(ops, cfg, np.arange(N, dtype=np.int32), False, m),
           "random": run(ops, cfg, np.arange(N, dtype=np.int32), True, m)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
