"""One config-3 block of the 4096-block batch: GPU (through the batch) vs oracle, with the
oracle's pivot margins (diagnostics).  usage: python tools/cfg3_block.py b"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

b = int(sys.argv[1])
nb = 4096
h = Handle(0)
s, t = synth.cauchy_params(0, nb)
Wt = synth.cauchy_blocks_torch(s, t, "cuda")
Ms = synth.multiplier_sparse_batch(0, nb, 512, 20)
bufs = pipeline.cur_batch(h, lra.Dense(Wt), lra.Multiplier(Ms), 16, 20, 2, nb)
torch.cuda.synchronize()
st = lra.stats_to_numpy(bufs.stats)[b]
Mb = dict(Ms, sp_row=Ms["sp_row"][b], sp_sign=Ms["sp_sign"][b])
W = synth.cauchy_block(s[b], t[b])
ora = O.cur_pipeline(W, Mb, 16, 20, 20, 2)
rho = float(np.sqrt(bufs.num2[b].item() / bufs.den2[b].item()))
print("I gpu", bufs.I[b].cpu().tolist())
print("I ora", list(ora.I))
print("J gpu", bufs.J[b].cpu().tolist())
print("J ora", list(ora.J))
print("rho gpu", rho, "ora", ora.rho, "rel", rho / ora.rho - 1)
print("gpu stats", st)
print("ora swaps", ora.ca.swaps, "lu", ora.ca.lu_steps, "loops", ora.ca.loops_done, "steps", ora.ca.steps)
print("ora min margin", ora.ca.min_pivot_margin, sorted(ora.ca.margins)[:5])
# the single-problem path on the same block
bufs1 = pipeline.cur(h, lra.Dense(Wt[b]), lra.Multiplier(Mb), 16, 20, 2)
torch.cuda.synchronize()
print("single-problem I equal oracle", bufs1.I.cpu().tolist() == list(ora.I),
      "rho", float(np.sqrt(bufs1.num2.item() / bufs1.den2.item())))
