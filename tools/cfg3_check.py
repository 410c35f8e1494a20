"""Config-3 batch through lra_batch at several batch sizes (diagnostics): status, a few blocks vs
the oracle.  usage: python tools/cfg3_check.py [nb ...]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

h = Handle(0)
for nb in [int(x) for x in sys.argv[1:]] or [148, 1024, 4096]:
    s, t = synth.cauchy_params(0, nb)
    Wt = synth.cauchy_blocks_torch(s, t, "cuda")
    Ms = synth.multiplier_sparse_batch(0, nb, 512, 20)
    bufs = pipeline.cur_batch(h, lra.Dense(Wt), lra.Multiplier(Ms), 16, 20, 2, nb)
    torch.cuda.synchronize()
    st = lra.stats_to_numpy(bufs.stats)
    rho = np.sqrt(bufs.num2.cpu().numpy() / bufs.den2.cpu().numpy())
    bad = 0
    for b in (0, nb // 2, nb - 1):
        ora = O.cur_pipeline(synth.cauchy_block(s[b], t[b]), dict(Ms, sp_row=Ms["sp_row"][b], sp_sign=Ms["sp_sign"][b]),
                             16, 20, 20, 2)
        bad += (list(bufs.I[b].cpu().numpy()) != list(ora.I)) or abs(rho[b] / ora.rho - 1) > 1e-4
    print(nb, "status ok", int(np.sum(st["status"] == 0)), "median rho", float(np.median(rho)), "bad", bad, flush=True)

# repeated calls on the overlapped schedule (side streams), then the profiled (serialized) one
nb = 4096
s, t = synth.cauchy_params(0, nb)
Wt = synth.cauchy_blocks_torch(s, t, "cuda")
Ms = synth.multiplier_sparse_batch(0, nb, 512, 20)
M = lra.Multiplier(Ms)
bufs = pipeline.BatchBuffers(nb, 16, 20)
import os
reps = int(os.environ.get("REPS", "6"))
for i in range(reps):
    pipeline.cur_batch(h, lra.Dense(Wt), M, 16, 20, 2, nb, bufs=bufs)
    if os.environ.get("SYNC_EACH"):
        torch.cuda.synchronize()
        ie = lra.debug_index_errors(reset=True)
        st = lra.stats_to_numpy(bufs.stats)
        I = bufs.I.cpu().numpy(); J = bufs.J.cpu().numpy()
        badI = np.nonzero((I < 0) | (I >= 512))[0]
        print("rep", i, "ok", ie, "bad I/J rows", len(badI), int(np.sum((J < 0) | (J >= 512))),
              "status!=0", int(np.sum(st["status"] != 0)), flush=True)
        if ie[0] or len(badI):
            print("   bad blocks", sorted(set((badI // 20).tolist()))[:10], "I sample", I.reshape(nb, 20)[badI[0] // 20] if len(badI) else None, flush=True)
torch.cuda.synchronize()
print("overlapped x", reps, "ok", flush=True)
h.profile(True)
pipeline.cur_batch(h, lra.Dense(Wt), M, 16, 20, 2, nb, bufs=bufs)
torch.cuda.synchronize()
print("profiled ok", h.profile_read(), flush=True)
h.profile(False)
