"""Planted-tie parity diagnostics (tests/test_gpu_parity.py::test_tie_rule_planted_ties_vs_oracle):
usage: python tools/tie_check.py cluster|grid|global [pairs_divisor]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import synth  # noqa: E402
from oracle import lra as O  # noqa: E402
from paper_1710_07946_b200 import Handle, lra, pipeline  # noqa: E402

tier = sys.argv[1]
div = int(sys.argv[2]) if len(sys.argv) > 2 else 8
if tier == "cluster":
    shape, r, k, d = (4096, 4096), 32, 48, 4
elif tier == "grid":
    shape, r, k, d = (9000, 600), 12, 16, 3
else:
    shape, r, k, d = (3000, 2600), 64, 96, 3
W = np.random.default_rng(30).standard_normal(shape)
pairs = {}
for axis, seed in ((0, 1), (1, 2)):
    g = np.random.default_rng(seed)
    n = W.shape[axis]
    perm = g.permutation(n)
    npairs = n // div
    for t, (a, b) in enumerate(zip(perm[:npairs], perm[npairs:2 * npairs])):
        f = 1.0 if t % 2 == 0 else 1.0 + 3e-13
        if axis == 0:
            W[b, :] = W[a, :] * f
        else:
            W[:, b] = W[:, a] * f
        pairs[(axis, int(b))] = (int(a), f)
W = np.asfortranarray(W)
mult = synth.multiplier_abridged(9, W.shape[1], d, k, "arht")
ora = O.cur_pipeline(W, mult, r, k, k, 3)
h = Handle(0)
lra.debug_counters(reset=True)
b = pipeline.cur(h, lra.Dense(lra.to_colmajor(W)), lra.Multiplier(mult), r, k, 3)
torch.cuda.synchronize()
c = lra.debug_counters(reset=True)
st = lra.stats_to_numpy(b.stats)[0]
I, J = b.I.cpu().tolist(), b.J.cpu().tolist()
print(tier, "exact rounds", c["exact_rounds"], "swaps gpu/ora", int(st["swaps"]), ora.ca.swaps,
      "lu", int(st["lu_steps"]), ora.ca.lu_steps, "loops", int(st["loops_done"]), ora.ca.loops_done)
for name, G, Ol, ax in (("I", I, list(ora.I), 0), ("J", J, list(ora.J), 1)):
    diffs = [(s, G[s], Ol[s]) for s in range(len(G)) if G[s] != Ol[s]]
    print(name, "mismatches", len(diffs))
    for s, gv, ov in diffs[:6]:
        print("   slot", s, "gpu", gv, "ora", ov, "gpu-pair", pairs.get((ax, gv)), "ora-pair", pairs.get((ax, ov)),
              "gpu src of", [k2 for k2, v in pairs.items() if k2[0] == ax and v[0] == gv][:2])
