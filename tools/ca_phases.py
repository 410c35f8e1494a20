"""Per-phase cycle counters of the C-A kernel on one config-2 matrix (diagnostics)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "arht"
W = synth.config2(0)
M = synth.multiplier_abridged(0, 4096, 4, 48, kind)
h = Handle(0)
Wd = lra.Dense(lra.to_colmajor(W))
Mm = lra.Multiplier(M)
bufs = pipeline.cur(h, Wd, Mm, 32, 48, 3)
torch.cuda.synchronize()
lra.debug_counters(reset=True)
h.profile(True)
bufs = pipeline.cur(h, Wd, Mm, 32, 48, 3, bufs=bufs)
torch.cuda.synchronize()
prof = h.profile_read()
cnt = lra.debug_counters(reset=True)
st = lra.stats_to_numpy(bufs.stats)[0]
out = {k: (v / 1965.0 if k not in ("pivot_steps", "nuc_sweeps", "nuc_rotations") else v) for k, v in cnt.items()}
print(json.dumps({"phases_us": out, "kernels_ms": prof, "swaps": int(st["swaps"]), "lu": int(st["lu_steps"])}, indent=1))
