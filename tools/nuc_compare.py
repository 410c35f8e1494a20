"""Bit-identity check of the nucleus pair loop against the reference loop (env LRA_NUC_OLD):
   python tools/nuc_compare.py OUT.npz   (run twice, with and without LRA_NUC_OLD=1)
   python tools/nuc_compare.py --cmp A.npz B.npz"""
import sys

import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print({"cases": len(a.files), "different": bad})
    sys.exit(1 if bad else 0)

import torch  # noqa: E402

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1710_07946_b200 import Handle, lra  # noqa: E402

h = Handle(0)
rng = np.random.default_rng(7)
out = {}
mats = {"cfg2": synth.config2(0), "cfg1": synth.config1(0),
        "cauchy": synth.cauchy_block(*[v[0] for v in synth.cauchy_params(0, 1)])}
cases = [("cfg2", 48, 48, 32), ("cfg2", 96, 96, 64), ("cfg2", 112, 112, 100), ("cfg2", 64, 128, 50), ("cfg2", 33, 33, 20),
         ("cfg2", 8, 13, 7), ("cfg2", 13, 8, 7), ("cfg2", 32, 48, 32), ("cfg1", 8, 8, 8), ("cauchy", 20, 20, 16)]
times = {}
ftimes = {}
for name, k, l, r in cases:
    W = mats[name]
    m, n = W.shape
    Wd = lra.Dense(lra.to_colmajor(W))
    for rep in range(3):
        I = torch.from_numpy(rng.choice(m, k, replace=False).astype(np.int64)).cuda()
        J = torch.from_numpy(rng.choice(n, l, replace=False).astype(np.int64)).cuda()
        U = torch.zeros((k, l), dtype=torch.float64, device="cuda")
        A = torch.zeros((r, m), dtype=torch.float64, device="cuda")
        B = torch.zeros((n, r), dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        h.profile(True)
        lra.lra_nucleus_factors(h, Wd, I, J, r, U, A, B, st)
        torch.cuda.synchronize()
        prof = h.profile_read()
        times[f"{name}_{k}x{l}"] = round(prof["k_nucleus"][0] * 1e3, 1)
        ftimes[f"{name}_{k}x{l}"] = (round(prof["k_factor_A"][0] * 1e3, 1), round(prof["k_factor_B"][0] * 1e3, 1))
        key = f"{name}_{k}_{l}_{r}_{rep}"
        out[key + "_U"] = U.cpu().numpy()
        out[key + "_A"] = A.cpu().numpy()
        out[key + "_B"] = B.cpu().numpy()
        out[key + "_st"] = st.cpu().numpy()
np.savez(sys.argv[1], **out)
print({"nucleus_us": times})
print({"factors_us": ftimes})
