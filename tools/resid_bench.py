"""Time the full a-posteriori pass alone (lra_cur_residual) on a config-2-sized fp32 matrix
with random fp64 factors (diagnostics).  usage: python tools/resid_bench.py [m] [n] [r] [prec]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
r = int(sys.argv[3]) if len(sys.argv) > 3 else 32
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 1
g = torch.Generator(device="cuda").manual_seed(0)
Wt = torch.randn((n, m), device="cuda", generator=g, dtype=torch.float32)
At = torch.randn((r, m), device="cuda", generator=g, dtype=torch.float64) * 1e-2
Bt = torch.randn((n, r), device="cuda", generator=g, dtype=torch.float64) * 1e-2
num2 = torch.empty(1, dtype=torch.float64, device="cuda")
den2 = torch.empty(1, dtype=torch.float64, device="cuda")
h = Handle(0)
W = lra.Dense(Wt)
for _ in range(3):
    lra.lra_cur_residual(h, W, At, Bt, r, num2, den2, prec=prec)
torch.cuda.synchronize()
lra.debug_counters_residual(reset=True)
lra.lra_cur_residual(h, W, At, Bt, r, num2, den2, prec=prec)
torch.cuda.synchronize()
c = lra.debug_counters_residual(reset=True)
nt = max(c["tiles"], 1)
print("per-tile cycles:", {k: round(v / nt) for k, v in c.items() if k != "tiles"}, "tiles", c["tiles"])
h.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
K = 20
for _ in range(K):
    lra.lra_cur_residual(h, W, At, Bt, r, num2, den2, prec=prec)
e1.record()
torch.cuda.synchronize()
prof = h.profile_read()
ms = e0.elapsed_time(e1) / K
print(f"m={m} n={n} r={r} prec={prec}: {ms*1e3:.1f} us/call, {m*n*4/ms/1e6:.0f} GB/s (W only)",
      {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.items()})
