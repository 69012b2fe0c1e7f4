"""Isolated DGEMM tile timings at the solver's shapes (run once with SCSF_TN_TMA=0 and once with 1).

  TN upper (Gram, unique entries n b (b + 1)) and full TN (2 n b1 b2) through scsf_gemm_tn, NN
  (2 n b1 b2) through scsf_gemm_nn; CUDA events over 20 calls after 3 warm-up calls.
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_23215_b200 import scsf  # noqa: E402

SHAPES = [("C2", 10000, 120), ("C3", 40000, 240), ("C4", 64000, 120), ("C5", 250000, 360)]


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
    out = {"tn_tma": os.environ.get("SCSF_TN_TMA", "1"), "rows": []}
    for name, n, b in SHAPES:
        ld = (n + 31) // 32 * 32
        X = torch.randn(b, ld, dtype=torch.float64, device="cuda")
        Y = torch.randn(b, ld, dtype=torch.float64, device="cuda")
        M = torch.randn(b, b, dtype=torch.float64, device="cuda")
        O = torch.empty_like(X)
        t_up = timeit(lambda: scsf.gemm_tn(X, X, n, upper=True))
        t_tn = timeit(lambda: scsf.gemm_tn(X, Y, n))
        t_nn = timeit(lambda: scsf.gemm_nn(X, M, n, out=O))
        row = {"config": name, "n": n, "b": b,
               "tn_upper_us": 1e3 * t_up, "tn_upper_tflops": n * b * (b + 1) / (t_up / 1e3) / 1e12,
               "tn_full_us": 1e3 * t_tn, "tn_full_tflops": 2.0 * n * b * b / (t_tn / 1e3) / 1e12,
               "nn_us": 1e3 * t_nn, "nn_tflops": 2.0 * n * b * b / (t_nn / 1e3) / 1e12}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
