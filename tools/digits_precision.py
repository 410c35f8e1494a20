"""Precision of the digit-slice reconstruction schemes of the tensor-core residual (DESIGN.md
§6.2), simulated exactly in numpy on the oracle's factors A, B:

  b128s6: balanced base-128 digits (|d| <= 64), S = 6 slices, levels s + u <= 5 (round 1 PRECISE)
  b128s3: the same with S = 3 (round 1 FAST)
  b256s5: balanced base-256 digits in [-128, 127] from X = rint(x 2^(8S)) (|x| < 127/256),
          S = 5, levels s + u <= 4, the last level rounded to 2^-8 of its weight (round 2 PRECISE)
  b256s4, b256s3: the same with S = 4 / 3 (S = 3 = round 2 FAST)

For each scheme: rho from the simulated product vs rho from the exact fp64 product (the
oracle's), relative difference; the C17 bar is 1e-4.  Exponents as the kernels: one per row of
A, one per 32-column tile of B.

usage: python tools/digits_precision.py [cfg2|cfg3|cfg5s]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402


def scale_exp(mx, base_bits):
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))).astype(np.int64) + 2, 0)
    if base_bits == 8:       # |x| < 127/256 so the top balanced digit stays in [-128, 127]
        x = mx * np.exp2(-e.astype(np.float64))
        e = np.where(x >= 127.0 / 256.0, e + 1, e)
    return e


def digits(x, S, base_bits):
    """x: array with |x| < 1/2 (base-128) or < 127/256 (base-256).  Returns list of S int arrays."""
    if base_bits == 7:
        y = x.copy()
        out = []
        for _ in range(S):
            y = y * 128.0
            q = np.rint(y)
            out.append(q.astype(np.int64))
            y = y - q
        return out
    X = np.rint(x * 2.0 ** (8 * S)).astype(np.int64)
    out = []
    for _ in range(S - 1):
        d = ((X + 128) & 255) - 128
        out.append(d)
        X = (X - d) >> 8
    out.append(X)
    assert np.all(np.abs(X) <= 128) and np.all(X <= 127)
    return out[::-1]                                   # most significant first


def recon(A, B, S, base_bits, last_round=False):
    m, r = A.shape
    n = B.shape[1]
    ea = scale_exp(np.abs(A).max(axis=1), base_bits)                    # per row
    colmax = np.abs(B).max(axis=0)
    tmax = np.array([colmax[j:j + 32].max() for j in range(0, n, 32)])
    fb = np.repeat(scale_exp(tmax, base_bits), 32)[:n]                  # per 32-column tile
    Ah = A * np.exp2(-ea)[:, None]
    Bh = B * np.exp2(-fb)[None, :]
    da, db = digits(Ah, S, base_bits), digits(Bh, S, base_bits)
    beta = 2.0 ** base_bits
    tot = np.zeros((m, n))
    for lev in range(S):
        P = np.zeros((m, n))
        for s in range(lev + 1):
            P += da[s].astype(np.float64) @ db[lev - s].astype(np.float64)   # exact (< 2^53)
        w = beta ** -(lev + 2)
        if last_round and lev == S - 1 and base_bits == 8:
            P = np.floor((P + 128) / 256) * 256
        tot += P * w
    return tot * np.exp2(ea)[:, None] * np.exp2(fb)[None, :]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cases = []
    if which == "cfg2":
        for seed in (0, 1):
            W = synth.config2(seed)
            res = O.cur_pipeline(W, synth.multiplier_abridged(0, 4096, 4, 48, "arht"), 32, 48, 48, 3)
            cases.append((f"cfg2 seed {seed}", W, res))
    elif which == "cfg3":
        s, t = synth.cauchy_params(0, 6)
        mult = synth.multiplier_sparse_batch(0, 6, 512, 20)
        for b in range(6):
            W = synth.cauchy_block(s[b], t[b])
            mb = dict(mult, sp_row=mult["sp_row"][b], sp_sign=mult["sp_sign"][b])
            cases.append((f"cfg3 block {b}", W, O.cur_pipeline(W, mb, 16, 20, 20, 2)))
    else:
        import torch
        Wt = synth.config5_torch(0, 8192, 8192, device="cpu")
        W = np.asfortranarray(Wt.numpy().T)
        cases.append(("cfg5 recipe 8192^2", W, O.cur_pipeline(W, synth.multiplier_abridged(0, 8192, 5, 96, "arht"),
                                                              64, 96, 96, 3)))
    for name, W, res in cases:
        W64 = np.asarray(W, dtype=np.float64)
        den = float(np.sum(W64 * W64))
        rho0 = np.sqrt(res.num2 / res.den2)
        line = [f"{name}: rho {rho0:.6e}"]
        for tag, S, bb, lr in (("b128s6", 6, 7, False), ("b128s3", 3, 7, False), ("b256s5", 5, 8, True),
                               ("b256s4", 4, 8, True), ("b256s3", 3, 8, True)):
            AB = recon(res.A, res.B, S, bb, lr)
            rho = np.sqrt(float(np.sum((W64 - AB) ** 2)) / den)
            line.append(f"{tag} {abs(rho / rho0 - 1):.1e}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
