"""One call of each hot kernel at a config's shapes, for `ncu --set full -k regex:...` captures.

  python tools/prof_kernels.py C3        # TN Gram (upper + full), NN rotation, streaming filter step
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    cfg = synth.get_config(name)
    n, b = cfg.n, cfg.b
    ld = (n + 31) // 32 * 32
    X = torch.randn(b, ld, dtype=torch.float64, device="cuda")
    Y = torch.randn(b, ld, dtype=torch.float64, device="cuda")
    M = torch.randn(b, b, dtype=torch.float64, device="cuda")
    O = torch.empty_like(X)
    f = synth.make_batch(cfg, 1)
    faces = [torch.from_numpy(x).cuda() for x in f.faces]
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).cuda())
    os.environ["SCSF_FILTER_STREAMING"] = "1"
    for _ in range(2):                        # warm-up pass, then the profiled pass
        scsf.gemm_tn(X, X, n, upper=True)
        scsf.gemm_tn(X, Y, n)
        scsf.gemm_nn(X, M, n, out=O)
        scsf.cheb_filter(ops, 0, X, 4, 1.0, 5e5, 4.9e5)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
