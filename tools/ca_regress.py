"""C-A regression fingerprint: runs lra_cross_approx / lra_batch on a fixed set of seeded
inputs and prints (I, J, stats with exact float hex of the certificates) as JSON, so two
builds of the C-A kernel can be compared bit for bit (diagnostics; not a parity test).

usage: python tools/ca_regress.py OUT.json"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402


def rec(bufs, nb=1):
    st = lra.stats_to_numpy(bufs.stats)
    out = []
    I = bufs.I.cpu().numpy().reshape(nb, -1)
    J = bufs.J.cpu().numpy().reshape(nb, -1)
    for b in range(nb):
        s = st[b]
        out.append({"I": [int(x) for x in I[b]], "J": [int(x) for x in J[b]],
                    "stats": [int(s[f]) for f in ("status", "loops_done", "lu_steps", "swaps", "cap_hits",
                                                  "sketch_swaps")],
                    "cert": [float(s["cert_rows"]).hex(), float(s["cert_cols"]).hex()]})
    return out


def main():
    h = Handle(0)
    res = {}
    for seed in range(4):
        W = synth.config1(seed)
        M = synth.multiplier_abridged(seed, 256, 3, 8, "arht")
        b = pipeline.cur(h, lra.Dense(lra.to_colmajor(W)), lra.Multiplier(M), 8, 8, 2)
        res[f"cfg1_s{seed}"] = rec(b)
    for seed in range(2):
        W = synth.config2(seed)
        Wd = lra.Dense(lra.to_colmajor(W))
        for kind in ("arht", "arft", "gaussian"):
            M = (synth.multiplier_gaussian(seed, 4096, 48) if kind == "gaussian"
                 else synth.multiplier_abridged(seed, 4096, 4, 48, kind))
            b = pipeline.cur(h, Wd, lra.Multiplier(M), 32, 48, 3)
            res[f"cfg2_{kind}_s{seed}"] = rec(b)
    nb = 64
    s, t = synth.cauchy_params(0, nb)
    Wt = synth.cauchy_blocks_torch(s, t, "cuda")
    Ms = synth.multiplier_sparse_batch(0, nb, 512, 20)
    b = pipeline.cur_batch(h, lra.Dense(Wt), lra.Multiplier(Ms), 16, 20, 2, nb)
    res["cfg3_64"] = rec(b, nb)
    for (m, n, d, k, r) in [(1000, 776, 3, 13, 9), (333, 520, 2, 7, 7), (130, 96, 5, 5, 3), (3000, 2048, 3, 64, 40),
                            (2048, 3000, 3, 33, 20)]:
        for dt in (np.float64, np.float32):
            W = np.asfortranarray(synth.factor_gaussian(m + n, m, n, r, 1e-14).astype(dt))
            M = synth.multiplier_abridged(7, n, d, k, "arht")
            b = pipeline.cur(h, lra.Dense(lra.to_colmajor(W)), lra.Multiplier(M), r, k, 3)
            res[f"rag_{m}x{n}_k{k}_{np.dtype(dt).name}"] = rec(b)
    c4 = synth.config4(0, m=8192, n=8192, p=16, dens_ab=0.05, dens_e=1e-3)
    A_t = torch.from_numpy(np.ascontiguousarray(c4["A"].T)).cuda()
    B_t = torch.from_numpy(np.ascontiguousarray(c4["B"].T)).cuda()
    rp, col, val = (torch.from_numpy(c4[x]).cuda() for x in ("row_ptr", "col", "val"))
    Wf = lra.Factored(A_t, B_t, rp, col, val, c4["m"], c4["n"], c4["p"])
    I0 = torch.from_numpy(synth.random_rows(0, c4["m"], 24)).cuda()
    bufs = pipeline.CurBuffers(c4["m"], c4["n"], 16, 24)
    lra.lra_cross_approx(h, Wf, None, I0, 16, 24, 24, 3, bufs.I, bufs.J, bufs.U, bufs.A, bufs.B, bufs.stats)
    torch.cuda.synchronize()
    res["cfg4_8192"] = rec(bufs)
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=0)
    print("cases", len(res))


if __name__ == "__main__":
    main()
