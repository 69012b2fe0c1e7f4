"""Per-phase time per operator with C concurrent chains (phase timers on): shows which phase
stretches under contention.   python tools/chain_phases.py [CFG] [N_OPS] [CHAINS...]"""
import resource
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    nops = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    chain_counts = [int(x) for x in sys.argv[3:]] or [1, 4, 16, 32]
    cfg = synth.get_config(name)
    f = synth.make_batch(cfg, nops)
    dev = torch.device("cuda", 0)
    params = torch.from_numpy(f.params).to(dev)
    if f.is_vib:
        ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
    else:
        faces = [torch.from_numpy(x).to(dev) for x in f.faces]
        ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
    perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    for C in chain_counts:
        for timing in (False, True):
            scsf.set_timing(timing)
            torch.cuda.synchronize()
            ru0 = resource.getrusage(resource.RUSAGE_SELF)
            t0 = time.perf_counter()
            _, _, st = scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=1,
                                         want_vecs=False, raise_on_fail=False)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            ru1 = resource.getrusage(resource.RUSAGE_SELF)
            cpu = (ru1.ru_utime - ru0.ru_utime) + (ru1.ru_stime - ru0.ru_stime)
            if not timing:
                rate = nops / dt
                cpu_frac = cpu / dt
                launches = scsf.launch_count()
                continue
            f_ms = np.mean([s["t_filter_ms"] for s in st])
            o_ms = np.mean([s["t_ortho_ms"] for s in st])
            r_ms = np.mean([s["t_rr_ms"] for s in st])
            per_op_chain = dt * 1e3 * C / nops
            print(f"{name} chains={C:3d}: {rate:7.1f} ops/s (untimed); per op per chain {per_op_chain:6.2f} ms: "
                  f"filter {f_ms:5.2f}  ortho {o_ms:5.2f}  rr {r_ms:5.2f}  other {per_op_chain - f_ms - o_ms - r_ms:5.2f}"
                  f"  | host cores busy {cpu_frac:4.1f}")
    scsf.set_timing(False)


if __name__ == "__main__":
    main()
