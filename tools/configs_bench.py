"""Per-configuration measurements of the hot path on one B200 (SURVEY §8(d) "report, per
config"): CUDA-event times per stage (lra_profile_*) and throughput, inputs resident in HBM.

  config 1  fp64 256², ARHT d=3, k=l=r=8, 2 sweeps: latency of one matrix (lra_preprocess +
            lra_cross_approx + lra_cur_residual) and throughput of lra_batch over 1184 seeds;
  config 2  fp32 4096², r=32, k=l=48, 3 sweeps: latency of one matrix per multiplier arm
            (ARHT, ARFT, Gaussian, quasi-Gaussian q=20);
  config 3  4096 Cauchy blocks 512² fp32 (4.29 GB), sparse ±1, r=16, k=l=20, 2 sweeps:
            blocks/s through lra_batch;
  config 4  W = A·B + E (65536², entry oracle, never formed), k=l=24, 3 sweeps from random
            rows, sampled residual on 1e6 pairs + exact factored norm.

usage: python tools/configs_bench.py [OUT.json]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

h = Handle(0)
out = {"gpu": torch.cuda.get_device_name(0)}


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    h.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    prof = h.profile_read()
    ms = e0.elapsed_time(e1) / reps
    return ms, {k: round(v[0] / reps * 1e3, 1) for k, v in prof.items()}


# ---------------------------------------------------------------- config 1
W1 = synth.config1(0)
M1 = lra.Multiplier(synth.multiplier_abridged(0, 256, 3, 8, "arht"))
W1d = lra.Dense(lra.to_colmajor(W1))
b1 = pipeline.CurBuffers(256, 256, 8, 8)
ms, st = timed(lambda: pipeline.cur(h, W1d, M1, 8, 8, 2, bufs=b1), 20)
nb1 = 1184
Wb = torch.from_numpy(np.ascontiguousarray(np.stack([synth.config1(s).T for s in range(nb1)]))).cuda()
bb1 = pipeline.BatchBuffers(nb1, 8, 8)
msb, stb = timed(lambda: pipeline.cur_batch(h, lra.Dense(Wb), M1, 8, 8, 2, nb1, bufs=bb1), 5)
rho1 = float(np.sqrt(b1.num2.item() / b1.den2.item()))
out["config1"] = {"latency_us": round(ms * 1e3, 1), "stages_us": st, "rho": rho1,
                  "batch": nb1, "batch_matrices_per_s": round(nb1 / (msb / 1e3), 1), "batch_stages_us": stb}
del Wb

# ---------------------------------------------------------------- config 2 arms
W2 = synth.config2(0)
W2d = lra.Dense(lra.to_colmajor(W2))
arms = {"arht": synth.multiplier_abridged(0, 4096, 4, 48, "arht"),
        "arft": synth.multiplier_abridged(0, 4096, 4, 48, "arft"),
        "gaussian": synth.multiplier_gaussian(0, 4096, 48),
        "qgauss_q20": synth.multiplier_qgauss(0, 4096, 20, 48)}
out["config2"] = {}
for name, mult in arms.items():
    M = lra.Multiplier(mult)
    b2 = pipeline.CurBuffers(4096, 4096, 32, 48, name == "arft")
    ms, st = timed(lambda: pipeline.cur(h, W2d, M, 32, 48, 3, bufs=b2), 5)
    out["config2"][name] = {"latency_us": round(ms * 1e3, 1), "stages_us": st,
                            "rho": float(np.sqrt(b2.num2.item() / b2.den2.item()))}

# ---------------------------------------------------------------- config 3
nb3 = 4096
s3, t3 = synth.cauchy_params(0, nb3)
W3 = synth.cauchy_blocks_torch(s3, t3, "cuda")
M3 = lra.Multiplier(synth.multiplier_sparse_batch(0, nb3, 512, 20))
bb3 = pipeline.BatchBuffers(nb3, 16, 20)
ms, st = timed(lambda: pipeline.cur_batch(h, lra.Dense(W3), M3, 16, 20, 2, nb3, bufs=bb3), 3)
rho3 = np.sqrt(bb3.num2.cpu().numpy() / bb3.den2.cpu().numpy())
out["config3"] = {"blocks": nb3, "ms_per_batch": round(ms, 3), "blocks_per_s": round(nb3 / (ms / 1e3), 1),
                  "input_GB": round(W3.numel() * 4 / 1e9, 2), "stages_us": st,
                  "rho_median": float(np.median(rho3)), "rho_max": float(rho3.max())}
del W3

# ---------------------------------------------------------------- config 4
t0 = time.time()
c4 = synth.config4(0)
gen_s = time.time() - t0
A_t = torch.from_numpy(np.ascontiguousarray(c4["A"].T)).cuda()
B_t = torch.from_numpy(np.ascontiguousarray(c4["B"].T)).cuda()
rp, col, val = (torch.from_numpy(c4[x]).cuda() for x in ("row_ptr", "col", "val"))
Wf = lra.Factored(A_t, B_t, rp, col, val, c4["m"], c4["n"], c4["p"])
I0 = torch.from_numpy(synth.random_rows(0, c4["m"], 24)).cuda()
ii, jj = (torch.from_numpy(x).cuda() for x in synth.sample_pairs(0, c4["m"], c4["n"], 1000000))
b4 = pipeline.CurBuffers(c4["m"], c4["n"], 16, 24)


def run4():
    lra.lra_cross_approx(h, Wf, None, I0, 16, 24, 24, 3, b4.I, b4.J, b4.U, b4.A, b4.B, b4.stats)
    lra.lra_cur_residual(h, Wf, b4.A, b4.B, 16, b4.num2, b4.den2, nsamples=1000000, si=ii, sj=jj)


ms, st = timed(run4, 3)
out["config4"] = {"ms": round(ms, 3), "stages_us": st, "gen_s": round(gen_s, 1),
                  "rho_sampled": float(np.sqrt(b4.num2.item() / b4.den2.item())),
                  "status": int(lra.stats_to_numpy(b4.stats)[0]["status"])}
js = json.dumps(out)
print(js)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(js + "\n")
