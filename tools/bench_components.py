"""Microbenchmark of libscsf component kernels at C2/C3/C5 shapes (CUDA events, warm)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_23215_b200 import scsf  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000.0   # us (includes the per-call sync of the ABI)


def main():
    out = {}
    rng = np.random.default_rng(0)
    for b in (120, 240):
        B = rng.standard_normal((b, b))
        dense = torch.from_numpy(B + B.T).cuda()
        d = np.sort(rng.uniform(30, 2000, b))
        E = rng.standard_normal((b, b)) * 1e-7 * d.max()
        warm = torch.from_numpy(np.diag(d) + E + E.T).cuda()
        for name, G in (("dense", dense), ("warm", warm)):
            th, Z, sw = scsf.syev_small(G, return_sweeps=True)
            out[f"syev_b{b}_{name}_us"] = timeit(lambda: scsf.syev_small(G))
            out[f"syev_b{b}_{name}_sweeps"] = sw
        Y = torch.randn(4 * b, b, dtype=torch.float64, device="cuda")
        S = (Y.T @ Y).contiguous()
        out[f"chol_inv_b{b}_us"] = timeit(lambda: scsf.chol_inv(S))
    for n, b in ((10000, 120), (40000, 240), (250000, 360)):
        ld = (n + 31) // 32 * 32
        X = torch.randn(b, ld, dtype=torch.float64, device="cuda")
        Y = torch.randn(b, ld, dtype=torch.float64, device="cuda")
        M = torch.randn(b, b, dtype=torch.float64, device="cuda")
        flops = 2.0 * n * b * b
        t = timeit(lambda: scsf.gemm_tn(X, Y, n))
        out[f"gemm_tn_n{n}_b{b}_us"] = t
        out[f"gemm_tn_n{n}_b{b}_tflops"] = flops / t / 1e6
        t = timeit(lambda: scsf.gemm_tn(X, X, n, upper=True))
        out[f"gemm_tn_upper_n{n}_b{b}_us"] = t
        if b <= 368:
            t = timeit(lambda: scsf.gemm_nn(X, M, n, out=Y))
            out[f"gemm_nn_n{n}_b{b}_us"] = t
            out[f"gemm_nn_n{n}_b{b}_tflops"] = flops / t / 1e6
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
