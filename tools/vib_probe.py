"""V1 (thin-plate vibration) convergence probe: per-operator iterations / residual / locked
count along the sorted queue, at the config's tol and max_iter (overridable).
  python tools/vib_probe.py [N] [chains] [max_iter] [tol]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = synth.get_config("V1")
    mi = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.max_iter
    tol = float(sys.argv[4]) if len(sys.argv) > 4 else cfg.tol
    f = synth.make_batch(cfg, N)
    params = torch.from_numpy(f.params).cuda()
    ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
    perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    ev, _, st = scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, cfg.degree, tol, mi, seed=3, want_vecs=False,
                                  raise_on_fail=False)
    starts = scsf.split_chains(len(perm), C)
    rows = [{"pos": k, "head": int(k in set(starts.tolist())), "it": s["iterations"], "status": s["status"],
             "locked": s["n_locked"], "resid": s["max_rel_resid"], "beta": s["beta"], "lam1": float(ev[k, 0]),
             "sweeps": s["jacobi_sweeps"]} for k, s in enumerate(st)]
    for r in rows:
        print(json.dumps(r))
    its = np.array([r["it"] for r in rows])
    print(json.dumps({"max_iter": mi, "tol": tol, "converged": int(sum(r["status"] == 0 for r in rows)),
                      "it_mean": float(its.mean()), "it_warm_mean": float(its[[not r["head"] for r in rows]].mean())}))


if __name__ == "__main__":
    main()
