"""HBM throughput of the full pre-processing pass W' = W D H_{n,d} P (lra_preprocess_full):
algorithmic bytes 2 m n s_e (read W once, write W' once).  usage: python tools/transform_bench.py [m] [d]"""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4
Wt = torch.randn((n, m), device="cuda", dtype=torch.float32)
Wp = torch.empty_like(Wt)
M = lra.Multiplier(synth.multiplier_abridged(0, n, d, n, "arht"))
h = Handle(0)
W = lra.Dense(Wt)
for _ in range(3):
    lra.lra_preprocess_full(h, W, M, Wp)
torch.cuda.synchronize()
h.profile(True)
K = 20
for _ in range(K):
    lra.lra_preprocess_full(h, W, M, Wp)
prof = h.profile_read()
ms = prof["k_transform_full"][0] / prof["k_transform_full"][1]
gbs = 2 * m * n * 4 / (ms * 1e-3) / 1e9
print(f"m=n={m} d={d}: k_transform_full {ms*1e3:.1f} us, {gbs:.0f} GB/s algorithmic (2 m n 4 B)")
