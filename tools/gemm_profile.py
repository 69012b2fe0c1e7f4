"""Per-kind DGEMM time and flops in one chain (phase timers on; SCSF_GEMM_PROFILE=1 makes the library
print one line per operator on stderr).  Kinds: 0 Gram (BCGS V_L^T F, CholQR Y^T Y), 1 triangular
R^-1 apply, 2 rotation, 3 dual Gram [Q1^T Q1 | Q1^T W1], 4 V <- Q1 M, 5 BCGS update F -= V_L C.

  SCSF_GEMM_PROFILE=1 python tools/gemm_profile.py C3 8 120 2> gp.err; python tools/gemm_profile.py --parse gp.err
"""
import json
import re
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--parse":
    tot_ms = [0.0] * 6
    tot_fl = [0.0] * 6
    for ln in open(sys.argv[2]):
        if not ln.startswith("scsf_gemm_profile"):
            continue
        for k, ms, fl in re.findall(r"k(\d)=([0-9.eE+-]+)/([0-9.eE+-]+)", ln):
            tot_ms[int(k)] += float(ms)
            tot_fl[int(k)] += float(fl)
    names = ["gram (BCGS / CholQR)", "triangular apply", "rotation", "dual Gram", "V <- Q1 M", "BCGS update"]
    out = {names[k]: {"ms": tot_ms[k], "gflop": tot_fl[k] / 1e9,
                      "tflops": (tot_fl[k] / (tot_ms[k] / 1e3) / 1e12) if tot_ms[k] > 0 else None} for k in range(6)}
    print(json.dumps(out, indent=1))
    sys.exit(0)

import torch  # noqa: E402

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
m = int(sys.argv[3]) if len(sys.argv) > 3 else 120
cfg = synth.get_config(name)
f = synth.make_batch(cfg, N)
faces = [torch.from_numpy(x).cuda() for x in f.faces]
ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).cuda())
params = torch.from_numpy(f.params).cuda()
perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
scsf.solve_queue(ops, perm[:2], cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, want_vecs=False)   # warm-up
scsf.set_timing(True)
scsf.solve_queue(ops, perm, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, want_vecs=False)
torch.cuda.synchronize()
print("done")
