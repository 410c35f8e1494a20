"""Per-phase C-A cycle counters of config 3 (512 x 512 Cauchy blocks, sparse sketch, k = l = 20,
2 sweeps) in ONE launch of B blocks (LRA_BATCH_GROUPS=1): microseconds per block of each phase
(summed over CTAs, so concurrent blocks add up), and the kernel times.
usage: LRA_BATCH_GROUPS=1 python tools/ca_phases_cfg3.py [B]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148
s, t = synth.cauchy_params(0, B)
Wt = synth.cauchy_blocks_torch(s, t, "cuda")
M = lra.Multiplier(synth.multiplier_sparse_batch(0, B, 512, 20))
h = Handle(0)
bufs = pipeline.cur_batch(h, lra.Dense(Wt), M, 16, 20, 2, B)
torch.cuda.synchronize()
lra.debug_counters(reset=True)
h.profile(True)
bufs = pipeline.cur_batch(h, lra.Dense(Wt), M, 16, 20, 2, B, bufs=bufs)
torch.cuda.synchronize()
prof = h.profile_read()
cnt = lra.debug_counters(reset=True)
out = {k: round(v / 1965.0 / B, 1) for k, v in cnt.items() if v}
print(json.dumps({"B": B, "phases_us_per_block": out, "kernels_ms": {k: round(v[0], 3) for k, v in prof.items()}}))
