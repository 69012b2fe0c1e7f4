"""Measure the fp64 GEMM peak on this GPU with cuBLAS (torch.matmul float64): burst and sustained."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = False
out = {}
for N in (4096, 8192):
    a = torch.randn(N, N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * N ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    out[f"dgemm_{N}_burst_tflops"] = best
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.time()
it = 0
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b)
    it += 1
    if it % 4 == 0:
        torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
out["dgemm_8192_sustained_tflops"] = it * 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
print(json.dumps(out))
