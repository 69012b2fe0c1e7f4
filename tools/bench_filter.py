"""Filter (Alg. 1) microbenchmark: scsf_cheb_filter on full-width blocks at the config shapes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    out = {}
    for name in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
        cfg = synth.get_config(name)
        f = synth.make_batch(cfg, 1)
        faces = [torch.from_numpy(x).cuda() for x in f.faces]
        ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).cuda())
        n, ld, b = cfg.n, ops.ld, cfg.b
        Y0 = torch.randn(b, ld, dtype=torch.float64, device="cuda")
        m = int(os.environ.get("BF_DEGREE", cfg.degree))
        for _ in range(2):
            scsf.cheb_filter(ops, 0, Y0, m, 30.0, 5e4, 4e4)
        torch.cuda.synchronize()
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            scsf.cheb_filter(ops, 0, Y0, m, 30.0, 5e4, 4e4)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byts = 16.0 * n * b + 24.0 * n * b * (m - 1) + 8.0 * (1 + cfg.dim) * n * m
        out[name] = {"n": n, "b": b, "m": m, "ms_per_filter": ms, "us_per_step": 1000 * ms / m,
                     "algorithmic_GBps": byts / (ms / 1e3) / 1e9, "frac_of_6547": byts / (ms / 1e3) / 1e9 / 6547.5}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
