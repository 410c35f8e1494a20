"""Tensor-core Gaussian sketch (reading C36) vs the oracle's fp64 sketch: max |Y_gpu - Y_ora|
relative to sum_j |W_ij| |Omega_jt|, on several shapes; plus device time of the launches."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

h = Handle(0)


def run(name, W, mult, reps=20):
    Wd = lra.Dense(lra.to_colmajor(W))
    M = lra.Multiplier(mult)
    m, n = W.shape
    lb = mult["lbar"]
    Y = torch.empty((lb, m), dtype=torch.float64, device="cuda")
    lra.lra_preprocess(h, Wd, M, Y)
    torch.cuda.synchronize()
    Yg = Y.cpu().numpy().T
    Yo = O.sketch(np.asarray(W, np.float64), mult)
    om = O.qgauss_omega(mult) if mult["kind"] == "qgauss" else np.asarray(mult["omega"], np.float64)
    bound = np.abs(np.asarray(W, np.float64)) @ np.abs(om)
    err = np.abs(Yg - Yo) / np.maximum(bound, 1e-300)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        lra.lra_preprocess(h, Wd, M, Y)
    ev1.record()
    torch.cuda.synchronize()
    us = ev0.elapsed_time(ev1) / reps * 1e3
    print(f"{name:28s} max rel-to-|W||Om| {err.max():.3e} (2^{np.log2(max(err.max(), 1e-300)):.1f})  "
          f"exact {np.array_equal(Yg, Yo)}  {us:8.1f} us/call", flush=True)
    return err.max()


g = np.random.default_rng(0)
run("cfg1 fp64 256 lb8", synth.config1(0), synth.multiplier_gaussian(0, 256, 8))
run("ragged fp32 1000x777 lb20", g.standard_normal((1000, 777)).astype(np.float32), synth.multiplier_gaussian(1, 777, 20))
run("ragged fp64 300x333 lb40", g.standard_normal((300, 333)), synth.multiplier_gaussian(2, 333, 40))
run("wide lb 100", g.standard_normal((700, 500)).astype(np.float32), synth.multiplier_gaussian(3, 500, 100))
run("cfg2 gaussian", synth.config2(0), synth.multiplier_gaussian(0, 4096, 48))
run("cfg2 qgauss q20", synth.config2(0), synth.multiplier_qgauss(0, 4096, 20, 48))
