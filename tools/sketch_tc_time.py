"""cfg2 Gaussian sketch through lra_preprocess, a few calls (for ncu launch lists)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

h = Handle(0)
W = synth.config2(0)
mult = synth.multiplier_gaussian(0, 4096, 48)
Wd = lra.Dense(lra.to_colmajor(W))
M = lra.Multiplier(mult)
Y = torch.empty((48, 4096), dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    lra.lra_preprocess(h, Wd, M, Y)
torch.cuda.synchronize()
print("ok")
