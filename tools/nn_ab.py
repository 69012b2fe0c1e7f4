"""Isolated NN products Out = X M at the solver's shapes: the library's NN kernel (run once with
SCSF_NN_TMA=0 -> k_gemm_nn3, once with 1 -> k_gemm_nn_tma) against cuBLAS DGEMM (torch.mm) on the
same operands; CUDA events over 20 calls after 3 warm-up calls.  Rows: (config, n, b1, b2) with
b1 = b2 = b (Rayleigh-Ritz rotation, CholQR apply) and b1 = L, b2 = nex-sized / half blocks
(BCGS against the locked columns)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_23215_b200 import scsf  # noqa: E402

SHAPES = [("C2", 10000, 120, 120), ("C3", 40000, 240, 240), ("C3", 40000, 200, 160), ("C4", 64000, 120, 120),
          ("C5", 250000, 360, 360), ("C5", 250000, 300, 180), ("C5/8", 31250, 360, 360)]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    out = {"nn_tma": os.environ.get("SCSF_NN_TMA", "1"), "rows": []}
    for name, n, b1, b2 in SHAPES:
        ld = (n + 31) // 32 * 32
        X = torch.randn(b1, ld, dtype=torch.float64, device="cuda")
        M = torch.randn(b2, b1, dtype=torch.float64, device="cuda")      # column-major b1 x b2
        O = torch.empty(b2, ld, dtype=torch.float64, device="cuda")
        t_nn = timeit(lambda: scsf.gemm_nn(X, M, n, out=O))
        Xn = X[:, :n].t()                                                 # n x b1 view (column-major)
        Mn = M.t()
        t_cb = timeit(lambda: torch.mm(Xn, Mn))
        ref = torch.mm(Xn, Mn)
        err = float((O[:, :n].t() - ref).abs().max() / ref.abs().max())
        f = 2.0 * n * b1 * b2
        row = {"config": name, "n": n, "b1": b1, "b2": b2, "nn_us": 1e3 * t_nn, "nn_tflops": f / (t_nn / 1e3) / 1e12,
               "cublas_us": 1e3 * t_cb, "cublas_tflops": f / (t_cb / 1e3) / 1e12, "ratio_vs_cublas": t_nn / t_cb,
               "max_rel_err": err}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
