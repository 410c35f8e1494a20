"""num2/den2 of the tensor-core residual through the fused split vs the two-kernel split
(run with and without LRA_SPLIT_OLD=1; prints the values as hex)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

h = Handle(0)
out = []
for (m, n, r, prec) in [(4096, 4096, 32, 1), (1000, 777, 17, 1), (4096, 4096, 64, 1), (1000, 3000, 48, 0), (300, 200, 5, 0)]:
    g = torch.Generator(device="cuda").manual_seed(m + n + r)
    Wt = torch.randn((n, m), device="cuda", generator=g, dtype=torch.float32)
    At = torch.randn((r, m), device="cuda", generator=g, dtype=torch.float64) * 1e-2
    Bt = torch.randn((n, r), device="cuda", generator=g, dtype=torch.float64) * 1e-2
    num2 = torch.empty(1, dtype=torch.float64, device="cuda")
    den2 = torch.empty(1, dtype=torch.float64, device="cuda")
    lra.lra_cur_residual(h, lra.Dense(Wt), At, Bt, r, num2, den2, prec=prec)
    torch.cuda.synchronize()
    out.append(f"{num2.item().hex()} {den2.item().hex()}")
print(" | ".join(out))
