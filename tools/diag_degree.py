"""Status of every operator of a C3 queue at a given degree (which ones fail, how)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402

name, N, C, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = synth.get_config(name)
f = synth.make_batch(cfg, N)
faces = [torch.from_numpy(x).cuda() for x in f.faces]
ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).cuda())
params = torch.from_numpy(f.params).cuda()
perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
_, _, st = scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=3, want_vecs=False,
                             raise_on_fail=False)
bad = [(k, s) for k, s in enumerate(st) if s["status"] != 0]
print(json.dumps({"m": m, "N": N, "failed": len(bad),
                  "examples": [{"pos": k, "status": s["status"], "iterations": s["iterations"], "n_locked": s["n_locked"],
                                "max_rel_resid": s["max_rel_resid"], "fallbacks": s["cholqr_fallbacks"],
                                "warm": s["warm"], "op": int(perm[k]), "filter_steps": s["filter_steps"]}
                               for k, s in bad[:8]],
                  "filter_steps": int(sum(s["filter_steps"] for s in st)),
                  "iterations": int(sum(s["iterations"] for s in st))}))
