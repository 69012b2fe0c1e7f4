"""A/B of the CUDA-graph replay on one config: run as two processes (SCSF_GRAPHS=0 / 1).

  SCSF_GRAPHS=1 python tools/graph_ab.py C3 64 32 20
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402

name, N, C, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = synth.get_config(name)
dev = torch.device("cuda", 0)
f = synth.make_batch(cfg, N)
params = torch.from_numpy(f.params).to(dev)
if f.is_vib:
    ops = scsf.assemble_vibration(cfg.nx, cfg.h, params)
else:
    faces = [torch.from_numpy(x).to(dev) for x in f.faces]
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
ws = scsf._workspace(scsf.solve_workspace(ops, cfg.L, cfg.nex).numel() * C, dev)
out = {"config": name, "N": N, "chains": C, "m": m, "graphs": os.environ.get("SCSF_GRAPHS", "1"),
       "bj_unroll": os.environ.get("SCSF_BJ_UNROLL", "0")}
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, _, st = scsf.solve_chains(ops, perm, C, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=3, want_vecs=False,
                                 raise_on_fail=False, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    its = sum(s["iterations"] for s in st)
    out[f"pass{rep}_ms"] = e0.elapsed_time(e1)
    out["iterations_total"] = its
    out["jacobi_sweeps_per_iteration"] = sum(s["jacobi_sweeps"] for s in st) / max(its, 1)
    out["converged"] = sum(s["status"] == 0 for s in st)
print(json.dumps(out), flush=True)
