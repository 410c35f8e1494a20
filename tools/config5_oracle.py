"""BASELINE config 5 at FULL size (131072^2 fp32 = 68.7 GB, generated on the device) checked
against the oracle ("full-size config 5"): the GPU hot path through the C-ABI, then
the fp64 oracle on the SAME bits, W never copied to host RAM as a whole:

  * sketch  Y = oracle.sketch on row slabs of W (the sketch is row-separable: Y[rows] depends
    on W[rows] only), slabs fetched from the device;
  * C-A     oracle.cross_approx on a lazy operand whose rows(I) / cols(J) / block(I, J) are
    gathered from the device tensor (fp32 -> fp64, exact);
  * nucleus / factors  oracle.canonical_nucleus, oracle.rank_r_factors;
  * residual  oracle.cur_residual on row slabs (num^2, den^2 summed in slab order).

Reports pivots (I, J, swaps, LU steps) GPU vs oracle, U (relative), rho (GPU PRECISE and FAST vs
the oracle), and the noise-floor explanation of rho > 1 (reading C15: N has variance 1e-8, so
||N||_F ~ 13.1 >> ||signal||_F ~ 2.25).  usage: python tools/config5_oracle.py [m] [out.json]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
out_path = sys.argv[2] if len(sys.argv) > 2 else None
r, k, d, T = 64, 96, 5, 3
SLAB = 2048
t0 = time.time()
U5, V5 = synth.config5_factors(0, m, n)
Wt = synth.config5_torch(0, m, n, factors=(U5, V5))        # (n, m): column-major m x n on device
torch.cuda.synchronize()
gen_s = time.time() - t0
mult = synth.multiplier_abridged(0, n, d, k, "arht")

# ---------------------------------------------------------------- GPU (C-ABI)
h = Handle(0)
W = lra.Dense(Wt)
M = lra.Multiplier(mult)
bufs = pipeline.CurBuffers(m, n, r, k)
t1 = time.time()
lra.lra_preprocess(h, W, M, bufs.Y)
lra.lra_cross_approx(h, W, bufs.Y, None, r, k, k, T, bufs.I, bufs.J, bufs.U, bufs.A, bufs.B, bufs.stats)
num2_p = torch.empty(1, dtype=torch.float64, device="cuda")
den2_p = torch.empty(1, dtype=torch.float64, device="cuda")
lra.lra_cur_residual(h, W, bufs.A, bufs.B, r, num2_p, den2_p, prec=lra.LRA_RECON_PRECISE)
lra.lra_cur_residual(h, W, bufs.A, bufs.B, r, bufs.num2, bufs.den2, prec=lra.LRA_RECON_FAST)
torch.cuda.synchronize()
gpu_s = time.time() - t1
st = lra.stats_to_numpy(bufs.stats)[0]
I_g, J_g = bufs.I.cpu().numpy(), bufs.J.cpu().numpy()
U_g = bufs.U.cpu().numpy().T
rho_prec = float(np.sqrt(num2_p.item() / den2_p.item()))
rho_fast = float(np.sqrt(bufs.num2.item() / bufs.den2.item()))
Yg = bufs.Y.cpu().numpy().T
del bufs


# ---------------------------------------------------------------- oracle on the same bits
def row_slab(i0, i1):
    return Wt[:, i0:i1].contiguous().cpu().numpy().T.astype(np.float64)   # (i1-i0, n)


class LazyDeviceOperand:
    """rows / cols / block of the device matrix, gathered on demand (exact fp32 -> fp64)."""
    m, n = m, n

    def rows(self, I):
        idx = torch.as_tensor(np.asarray(I, np.int64), device="cuda")
        return Wt[:, idx].cpu().numpy().T.astype(np.float64)

    def cols(self, J):
        idx = torch.as_tensor(np.asarray(J, np.int64), device="cuda")
        return Wt[idx, :].cpu().numpy().T.astype(np.float64)

    def block(self, I, J):
        return self.cols(J)[np.asarray(I, np.int64), :]


t2 = time.time()
Y = np.empty((m, k))
for i0 in range(0, m, SLAB):
    Y[i0:i0 + SLAB] = O.sketch(row_slab(i0, i0 + SLAB), mult)
sketch_exact = bool(np.array_equal(Y, Yg))
op = LazyDeviceOperand()
ca = O.cross_approx(op, k, k, T, Y=Y)
Uo, Sr, sr, Tr = O.canonical_nucleus(op.block(ca.I, ca.J), r)
A, B = O.rank_r_factors(op.cols(ca.J), op.rows(ca.I), Sr, sr, Tr)
num2 = den2 = 0.0
for i0 in range(0, m, SLAB):
    a_, b_ = O.cur_residual(row_slab(i0, i0 + SLAB), A[i0:i0 + SLAB], B)
    num2 += a_
    den2 += b_
rho_o = float(np.sqrt(num2 / den2))
ora_s = time.time() - t2
# the noise floor (reading C15): ||N||_F from the signal part  U diag(s) V^T  (exact Gram form)
sig = synth.config5_sigma(64)
signal_F = float(np.sqrt(np.sum(sig ** 2)))
out = {"config": f"cfg5 {m}x{n} fp32, r={r}, k=l={k}, ARHT d={d}, {T} sweeps",
       "gen_s": round(gen_s, 1), "gpu_s": round(gpu_s, 2), "oracle_s": round(ora_s, 1),
       "sketch_bit_exact": sketch_exact,
       "I_equal": bool(np.array_equal(I_g, ca.I)), "J_equal": bool(np.array_equal(J_g, ca.J)),
       "swaps_gpu": int(st["swaps"]), "swaps_oracle": int(ca.swaps),
       "lu_gpu": int(st["lu_steps"]), "lu_oracle": int(ca.lu_steps),
       "loops_gpu": int(st["loops_done"]), "loops_oracle": int(ca.loops_done),
       "U_rel_err": float(np.max(np.abs(U_g - Uo)) / np.max(np.abs(Uo))),
       "rho_oracle": rho_o, "rho_gpu_precise": rho_prec, "rho_gpu_fast": rho_fast,
       "rho_rel_err_precise": abs(rho_prec / rho_o - 1), "rho_rel_err_fast": abs(rho_fast / rho_o - 1),
       "norm_W_F": float(np.sqrt(den2)), "norm_signal_F": signal_F,
       "noise_F_expected": float(np.sqrt(m * n * 1e-8)),
       "note": "rho > 1 is the oracle's own value: the recipe is noise-dominated (reading C15, N ~ N(0, 1e-8)); "
               "a CUR whose generator is mostly noise amplifies the noise rows/columns it copies"}
print(json.dumps(out))
if out_path:
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
