"""One warm-start chain of a config (default C2, 6 operators) for ncu launch lists / captures.

  python tools/profile_chain.py [CFG] [N_OPS] [CHAINS] [DEGREE]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    nops = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    chains = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    cfg = synth.get_config(name)
    m = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.degree
    f = synth.make_batch(cfg, nops)
    dev = torch.device("cuda", 0)
    params = torch.from_numpy(f.params).to(dev)
    if f.is_vib:
        ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
    else:
        faces = [torch.from_numpy(x).to(dev) for x in f.faces]
        ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
    perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if chains == 1:
        ev, _, st = scsf.solve_queue(ops, perm, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=1,
                                     want_vecs=False, raise_on_fail=False)
    else:
        ev, _, st = scsf.solve_chains(ops, perm, chains, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter,
                                      seed=1, want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = [s["iterations"] for s in st]
    print(f"{name}: {nops} ops in {dt*1e3:.1f} ms, iterations {its}, status {[s['status'] for s in st]}, "
          f"launches {scsf.launch_count()}")


if __name__ == "__main__":
    main()
