"""The row-sharded decomposition of the hot path, checked on CPU with
world_size-2 and -3 gloo process groups against the single-process oracle.  Each rank holds the
rows [g cm, g cm + m_g) of W (cm = ceil(m / G), the standard split).  Exactly as liblra.so's
sharded path does with NCCL:
  * the blocks whose rows are W's rows (the sketch Y, W[:,J]) are assembled by an ALL-GATHER
    of equal chunks (local rows packed, zero-padded to cm rows) and an unpack;
  * the blocks with data-dependent ownership (W[I,:]^T, W[I,J]) by an all-reduce SUM of
    owner-scattered rows into zeroed buffers (exact: x + 0 = x);
  * the maxvol runs replicated; the early exit (reading C13) is decided from the replicated
    swap counts (the library evaluates it on the device);
  * the residual is the sum of the ranks' partial norms.
Test infrastructure only (uses oracle/)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import lra as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sum(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy()


def _gather_rows(local, cm, m, ws):
    """local: (m_g, q) rows of this rank -> (m, q) assembled: every rank packs a cm x q chunk
    (zero rows beyond m_g), all_gather, unpack rank g's chunk into rows g cm .. (k_pack_rows,
    NCCL all-gather, k_unpack_chunks)."""
    q = local.shape[1]
    chunk = np.zeros((cm, q))
    chunk[:local.shape[0]] = local
    parts = [torch.zeros((cm, q), dtype=torch.float64) for _ in range(ws)]
    dist.all_gather(parts, torch.from_numpy(chunk))
    out = np.concatenate([p.numpy() for p in parts], axis=0)
    return out[:m]


def _worker(rank, ws, port, W, mult, r, k, sweeps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    m, n = W.shape
    cm = -(-m // ws)
    row0, row1 = rank * cm, min(m, (rank + 1) * cm)
    Wl = W[row0:row1]
    # stage 1: local sketch rows (Y = W M is row-local) -> assembled Y (all-gather)
    Y = _gather_rows(O.sketch(Wl, mult), cm, m, ws)
    I = O.maxvol(Y).S
    J = None
    steps = []
    for loop in range(sweeps):
        Rt = np.zeros((n, k))                   # W[I,:]^T from the rows this rank owns
        for s, i in enumerate(I):
            if row0 <= i < row1:
                Rt[:, s] = Wl[i - row0]
        Rt = _sum(Rt)
        rh = O.maxvol(Rt, J)
        Cb = _gather_rows(Wl[:, rh.S], cm, m, ws)          # W[:,J] (all-gather)
        rv = O.maxvol(Cb, I)
        J, I = rh.S, rv.S
        steps += [rh.swaps, rv.swaps]
        if loop > 0 and rh.swaps == 0 and rv.swaps == 0:
            break
    G = np.zeros((k, k))
    for s, i in enumerate(I):
        if row0 <= i < row1:
            G[s] = Wl[i - row0, J]
    G = _sum(G)
    Rt = np.zeros((n, k))
    for s, i in enumerate(I):
        if row0 <= i < row1:
            Rt[:, s] = Wl[i - row0]
    Rt = _sum(Rt)
    U, Sr, sr, Tr = O.canonical_nucleus(G, r)
    A_loc, B = O.rank_r_factors(Wl[:, J], Rt.T, Sr, sr, Tr)
    num, den = O.cur_residual(Wl, A_loc, B)
    num, den = _sum(np.array([num, den]))
    out[rank] = {"I": [int(x) for x in I], "J": [int(x) for x in J], "U": U, "num2": float(num),
                 "den2": float(den), "steps": steps}
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_row_sharded_protocol_equals_oracle(ws):
    W = synth.factor_gaussian(4, 600, 512, 6, 1e-8)
    mult = synth.multiplier_abridged(4, 512, 3, 8, "arht")
    ora = O.cur_pipeline(W, mult, 6, 8, 8, 3)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(ws, port, W, mult, 6, 8, 3, out), nprocs=ws, start_method="spawn")
    for rk in range(ws):
        res = out[rk]
        assert res["I"] == list(ora.I) and res["J"] == list(ora.J)          # replicated pivots
        assert np.array_equal(res["U"], ora.U)                               # same G bits -> same U
        assert res["den2"] == pytest.approx(ora.den2, rel=1e-14)
        rho = np.sqrt(res["num2"] / res["den2"])
        assert abs(rho - ora.rho) <= 1e-12 * 10 + 1e-9 * ora.rho
    assert out[0]["num2"] == out[ws - 1]["num2"]                            # identical on every rank
