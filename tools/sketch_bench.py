"""Time lra_preprocess (stage 1 of Alg 10.2) on a config-2-sized fp32 matrix for every
multiplier kind (diagnostics): us per call, the per-kernel split, and the algorithmic rate
(HBM bytes for the structured kinds, fp64 FLOP/s for the dense ones).
usage: python tools/sketch_bench.py [n] [lbar]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
lbar = int(sys.argv[2]) if len(sys.argv) > 2 else 48
g = torch.Generator(device="cuda").manual_seed(0)
Wt = torch.randn((n, n), device="cuda", generator=g, dtype=torch.float32)
W = lra.Dense(Wt)
h = Handle(0)
kinds = {"arht": synth.multiplier_abridged(0, n, 4, lbar, "arht"),
         "arft": synth.multiplier_abridged(0, n, 4, lbar, "arft"),
         "sparse": synth.multiplier_sparse(0, n, lbar),
         "gaussian": synth.multiplier_gaussian(0, n, lbar),
         "qgauss_q20": synth.multiplier_qgauss(0, n, 20, lbar)}
out = {}
for name, mult in kinds.items():
    M = lra.Multiplier(mult)
    Y = torch.empty((lbar, n, 2) if name == "arft" else (lbar, n), dtype=torch.float64, device="cuda")
    for _ in range(3):
        lra.lra_preprocess(h, W, M, Y)
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record()
    for _ in range(K):
        lra.lra_preprocess(h, W, M, Y)
    e1.record()
    torch.cuda.synchronize()
    prof = h.profile_read()
    us = e0.elapsed_time(e1) / K * 1e3
    rec = {"us_per_call": round(us, 1), "kernels_us": {k: round(v[0] / v[1] * 1e3, 1) for k, v in prof.items()}}
    if name in ("gaussian", "qgauss_q20"):
        rec["fp64_gflops"] = round(2.0 * n * n * lbar / (us * 1e-6) / 1e9, 1)
    else:
        d = 4
        fib = len(set(int(c) % (n >> d) for c in mult["col"])) if name != "sparse" else None
        byts = (fib * (1 << d) * n * 4 if fib else lbar * 4 * n * 4) + n * lbar * 8
        rec["algorithmic_GBs"] = round(byts / (us * 1e-6) / 1e9, 1)
    out[name] = rec
print(json.dumps(out))
