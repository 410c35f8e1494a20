"""Per-phase C-A cycle counters averaged over a batch of B config-2 matrices in ONE launch
(LRA_BATCH_GROUPS=1) — compare with tools/ca_phases.py (one matrix) to see how concurrency
changes each phase.  usage: LRA_BATCH_GROUPS=1 python tools/ca_phases_batch.py [B]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
Ws = np.stack([synth.config2(s).T for s in range(B)]).astype(np.float32)
Wt = torch.from_numpy(np.ascontiguousarray(Ws)).cuda()
M = lra.Multiplier(synth.multiplier_abridged(0, 4096, 4, 48, "arht"))
h = Handle(0)
bufs = pipeline.cur_batch(h, lra.Dense(Wt), M, 32, 48, 3, B)
torch.cuda.synchronize()
lra.debug_counters(reset=True)
h.profile(True)
bufs = pipeline.cur_batch(h, lra.Dense(Wt), M, 32, 48, 3, B, bufs=bufs)
torch.cuda.synchronize()
prof = h.profile_read()
cnt = lra.debug_counters(reset=True)
st = lra.stats_to_numpy(bufs.stats)
out = {k: round(v / 1965.0 / B, 1) for k, v in cnt.items() if v and k != "pivot_steps"}
print(json.dumps({"B": B, "phases_us_per_matrix": out, "kernels_ms": {k: round(v[0], 3) for k, v in prof.items()},
                  "swaps": st["swaps"].tolist()}))
