"""Measure the FP64 roofline denominator on this B200: cuBLAS DGEMM 8192^3 (best of 10) and a
DFMA-chain kernel is not needed — the library GEMM is the reference, like MEASURED_PEAKS.json's
bf16 figure.  Prints one JSON line."""
import json

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"fp64_dgemm_tflops": 2 * n ** 3 / (best / 1e3) / 1e12, "n": n, "ms": best}))
