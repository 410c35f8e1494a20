#!/usr/bin/env python
"""bench.py — throughput of the superfast-CUR hot path on B200 (BASELINE.json metric:
"CUR LRA matrices/sec and preprocess+residual GB/s vs HBM peak, 1/2/4/8 B200").

Headline (default, ``--workload cfg2``): one step = the whole hot path (§8(a): sketch, C-A
sweeps, nucleus + factors, full a-posteriori check) over one batch of B synthetic config-2
matrices per GPU (W = U·diag(σ)·Vᵀ fp32 4096², r = 32, k = l = 48, ARHT d = 4, 3 sweeps)
through ``lra_batch``.  Two batches alternate, so consecutive steps never find their inputs in
L2 (2·B·67 MB > 126 MB).  N > 1: one process per GPU, independent matrices per rank, no
collective on the data path ("weak"), max-over-ranks device time.

Measurement protocol (VERDICT r1 "make the measurement honest"):
  * the headline region runs with kernel profiling OFF (the overlapped schedule as shipped);
  * an ISOLATION pass then replays the same batches with profiling on: lra_batch runs its
    groups in order on one stream and every kernel is bracketed by events on its launch
    stream, so each kernel's interval is its own device time (Σ kernel ms ≤ the isolated
    step); ``roofline`` and ``stage_rooflines`` are computed from those device times;
  * secondary workloads in the same line (``workloads``): config 5 (131072² fp32 = 68.7 GB,
    row-sharded over the N ranks, each rank generating its shard on device) with the
    preprocess and residual GB/s the metric names, and config 3 (4096 Cauchy blocks dealt
    out across ranks) in blocks/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--workload cfg2|cfg5|cfg3]
                  [--impl native|reference] [--no-extra] [--no-e2e] [--no-cpu-baseline]
  N > 1 without WORLD_SIZE in the environment: bench.py starts N ranks itself through
  torch.distributed.run (127.0.0.1).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---------------------------------------------------------------- workload definitions
M_ROWS = N_COLS = 4096
R, K, SWEEPS, DEPTH = 32, 48, 3, 4
WORKLOAD = (f"cfg2-arht: W=U*diag(s)*V^T fp32 {M_ROWS}x{N_COLS}, s_i=1 (i<=32) then 1e-6*0.9^(i-32); "
            f"r={R}, k=l={K}, ARHT d={DEPTH} +-1 diagonal, {SWEEPS} C-A sweeps, full residual (PRECISE)")
METRIC = "CUR LRA matrices/sec (config 2, ARHT) — sketch+C-A+nucleus+residual"

C5_M = C5_N = 131072
C5_R, C5_K, C5_D, C5_T = 64, 96, 5, 3
C5_WORKLOAD = (f"cfg5: W=U*diag(s)*V^T+N fp32 {C5_M}x{C5_N} (68.7 GB) row-sharded, s_i=10^(-3(i-1)/63), "
               f"N~N(0,1e-8); r={C5_R}, k=l={C5_K}, ARHT d={C5_D}, {C5_T} sweeps, full residual (FAST)")
C5_METRIC = "CUR LRA matrices/sec (config 5, 131072^2 row-sharded) — sketch+C-A+nucleus+residual"

C3_NB, C3_M, C3_R, C3_K, C3_T = 4096, 512, 16, 20, 2
C3_WORKLOAD = (f"cfg3: {C3_NB} Cauchy blocks W_ij=fl32(1/(s_i-t_j)) {C3_M}x{C3_M}, s~U[0,1], t~U[2,3]; "
               f"sparse +-1 (4/col), r={C3_R}, k=l={C3_K}, {C3_T} sweeps, full residual (PRECISE); blocks dealt to ranks")
C3_METRIC = "CUR LRA blocks/sec (config 3, FMM Cauchy blocks) — sketch+C-A+nucleus+residual"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(args_in):
    """--gpus N > 1 outside torchrun: start N ranks (one process per GPU) and wait."""
    n = args_in.gpus
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


class Clocks:
    """nvidia-smi sampler (10 ms) for the clocks line of the JSON; started before the warm-up and
    awaited (ready) so that its first sample precedes the timed region."""

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "10"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.t0 = self.t1 = None

    def ready(self, timeout=10.0):
        """Block until nvidia-smi has written its first sample (its start-up takes ~0.1-1 s)."""
        if self.p is None:
            return
        t = time.time()
        while time.time() - t < timeout:
            try:
                if os.path.getsize(self.f.name) > 0:
                    return
            except OSError:
                pass
            time.sleep(0.01)

    def window(self, t0, t1):
        self.t0, self.t1 = t0, t1

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows, all_rows = [], []
        import datetime
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                row = (float(parts[1]), float(parts[2]), parts[5:9])
            except ValueError:
                continue
            all_rows.append(row)
            try:   # keep the samples taken inside the timed window
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if self.t0 is None or ts is None or (self.t0 - 0.01 <= ts <= self.t1 + 0.01):
                rows.append(row)
        if not rows:
            rows = all_rows
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [r[0] for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def _oracle_cores():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((d.get("num_threads", 1) for d in info), default=1)
        return int(n)
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- reference arm (the oracle)
def _oracle_cfg2(n_mats, seed0):
    import synth
    from oracle import lra as O
    mult = synth.multiplier_abridged(0, N_COLS, DEPTH, K, "arht")
    Ws = [synth.config2(seed0 + i, n=N_COLS) for i in range(n_mats)]
    t = time.perf_counter()
    for W in Ws:
        O.cur_pipeline(W, mult, R, K, K, SWEEPS)
    return time.perf_counter() - t


def _oracle_cfg3(n_blocks, seed):
    import synth
    from oracle import lra as O
    s, t = synth.cauchy_params(seed, n_blocks, C3_M, C3_M)
    mult = synth.multiplier_sparse_batch(seed, n_blocks, C3_M, C3_K)
    Ws = [synth.cauchy_block(s[b], t[b]) for b in range(n_blocks)]
    t0 = time.perf_counter()
    for b in range(n_blocks):
        mb = dict(mult, sp_row=mult["sp_row"][b], sp_sign=mult["sp_sign"][b])
        O.cur_pipeline(Ws[b], mb, C3_R, C3_K, C3_K, C3_T)
    return time.perf_counter() - t0


def cpu_baseline(n_mats=4):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload."""
    dt = _oracle_cfg2(n_mats, 90000)
    return {"value": n_mats / dt, "unit": "matrices/s", "cores": _oracle_cores(), "kind": "oracle",
            "sample": f"{n_mats} config-2 matrices (full size) through oracle.cur_pipeline, {dt:.1f} s"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    cores = _oracle_cores()
    if args.workload == "cfg5":
        print(json.dumps({"impl": "reference", "unavailable": "the fp64 oracle needs the 68.7 GB config-5 matrix in "
                          "host RAM and hours per step; the reference arm runs cfg2 / cfg3"}), flush=True)
        return
    if args.workload == "cfg3":
        nb = 8
        for _ in range(args.warmup):
            _oracle_cfg3(1, 7)
        dts = [_oracle_cfg3(nb, 100 + i) for i in range(args.steps)]
        v = nb * args.steps / sum(dts)
        metric, unit, wl, sample = C3_METRIC, "blocks/s", C3_WORKLOAD, f"{nb} config-3 blocks per step"
    else:
        for i in range(args.warmup):
            _oracle_cfg2(1, 70000 + i)
        dts = [_oracle_cfg2(1, 80000 + i) for i in range(args.steps)]
        v = args.steps / sum(dts)
        metric, unit, wl, sample = METRIC, "matrices/s", WORKLOAD, "1 full-size config-2 matrix per step"
    line = {"impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(dts) / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl,
                                           "note": "reference arm = the fp64 numpy oracle (no reference code exists)"},
            "cpu_baseline": {"value": v, "unit": unit, "cores": cores, "kind": "oracle",
                             "sample": f"{sample}, {args.steps} steps"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- algorithmic bytes
def _fibers(mult, n, d):
    s = n >> d
    return len({int(c) % s for c in mult["col"]})


def alg_bytes_cfg2(name, mult, mats, loops=SWEEPS):
    """Algorithmic bytes of `name` over `mats` config-2 matrices (what the method must move)."""
    m, n = M_ROWS, N_COLS
    if name.startswith("k_sketch"):
        return mats * (m * (1 << DEPTH) * _fibers(mult, n, DEPTH) * 4 + m * K * 8)
    if name == "k_residual_tc":
        return mats * m * n * 4
    if name == "residual_stage":      # split + tensor-core pass + reduce: W once, A and B once
        return mats * (m * n * 4 + (m * R + R * n) * 8)
    if name == "k_ca":                # Y block + per loop W[I,:] and W[:,J] (SURVEY §8(d) gathers)
        return mats * (m * K * 8 + loops * (K * n + m * K) * 4)
    return 0


def _roof(name, byts, ms_per_launch, peaks, src):
    ach = byts / (ms_per_launch * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": ach / peaks["hbm_gbs"], "peak_source": src, "traffic": None,
            "ms_per_launch": ms_per_launch}


def _ncu_traffic(kname, mats_per_launch):
    """dram read+write bytes per launch of kname from the newest committed ncu --set full summary
    (profiles/<round>/ncu_full*.txt), scaled to mats_per_launch."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_full_final.txt")))
    key = {"k_ca": "k_cacl", "k_residual_tc": "k_resid<"}.get(kname, kname)

    def val(x):
        x = x.strip()
        f = float(x.split()[0])
        return f * (1e9 if "Gbyte" in x else 1e6 if "Mbyte" in x else 1e3 if "Kbyte" in x else 1)

    for path in reversed(files):
        for line in open(path):
            if not line.startswith("Kernel Name=") or key not in line.split(";")[0]:
                continue
            f = dict(kv.split("=", 1) for kv in (x.strip() for x in line.split(";")) if "=" in kv)
            rd, wr = val(f["dram__bytes_read.sum"]), val(f["dram__bytes_write.sum"])
            mats = f.get("matrices_per_launch")
            if mats is None:
                grid = int(re.sub(r"[^0-9]", "", f.get("launch__grid_size", "0")) or 0)
                cdim = int(re.sub(r"[^0-9]", "", f.get("launch__cluster_dim_x", "0")) or 0)
                if key == "k_cacl" and grid and cdim:
                    mats = grid / cdim
                elif key.startswith("k_residual"):
                    mats = rd / (M_ROWS * N_COLS * 4)
                else:
                    return None
            return {"bytes_per_launch": (rd + wr) / float(mats) * mats_per_launch,
                    "source": os.path.relpath(path, ROOT)}
    return None


def _gen_batch(seeds):
    import synth
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        Ws = list(ex.map(lambda s: synth.config2(s, n=N_COLS), seeds))
    out = np.empty((len(seeds), N_COLS, M_ROWS), dtype=np.float32)
    for i, W in enumerate(Ws):
        out[i] = W.T
    return out


def _max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _timed(fn, steps, ws, st, streams=()):
    """steps calls of fn bracketed by a barrier + synchronize, CUDA events on stream st (the other
    streams fn launches on wait for the start event; the end event waits for all of them); max
    over ranks."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    others = [s for s in streams if s != st]
    for s in others:
        s.wait_event(e0)
    for i in range(steps):
        fn(i)
    for s in others:
        ev = torch.cuda.Event()
        ev.record(s)
        st.wait_event(ev)
    e1.record(st)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    return _max_over_ranks(e0.elapsed_time(e1), ws)


def _isolated(h, fn, steps, ws):
    """Isolation pass: profiling on (lra_batch groups serialized on one stream, an event pair
    per kernel on its launch stream).  Returns ({kernel: (ms per step, launches per step)},
    isolated ms per step)."""
    import torch
    torch.cuda.synchronize()
    h.profile(True)
    t = _timed(fn, steps, 1, torch.cuda.current_stream())
    prof = h.profile_read()
    h.profile(False)
    return {k: (v[0] / steps, v[1] / steps) for k, v in prof.items()}, t / steps


# ---------------------------------------------------------------- secondary workloads
def run_sketch_tc(h, peaks, src, reps=20):
    """The config-2 Gaussian sketch Y = W Omega (4096^2 fp32, lbar = 48) on the tensor cores
    (sketch_tc.cu, reading C36): device time per call (events), per-kernel split (isolation), and
    the tensor roofline of k_sketch_tc: int8 MACs issued (28 digit-slice products of M = 128,
    N = 48, K = 32 per 128-row tile and K-step) over its launch time, against the int8 dense peak
    = 2 x the measured bf16 peak (the guide's nominal ratio)."""
    import torch
    import synth
    from paper_1710_07946_b200 import lra
    W = torch.from_numpy(np.ascontiguousarray(synth.config2(0).T)).cuda()     # (n, m): column-major m x n
    Wd = lra.Dense(W)
    M = lra.Multiplier(synth.multiplier_gaussian(0, N_COLS, K))
    Y = torch.empty((K, M_ROWS), dtype=torch.float64, device="cuda")
    for _ in range(3):
        lra.lra_preprocess(h, Wd, M, Y)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        lra.lra_preprocess(h, Wd, M, Y)
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    prof, _ = _isolated(h, lambda i: lra.lra_preprocess(h, Wd, M, Y), reps, 1)
    main_ms = prof.get("k_sketch_tc", (float("nan"), 1))[0]
    tiles, ksteps = (M_ROWS + 127) // 128, (N_COLS + 31) // 32
    macs = tiles * ksteps * 28 * 128 * 48 * 32
    ach = 2.0 * macs / (main_ms * 1e-3) / 1e12
    peak = 2.0 * peaks.get("bf16_tflops", 1590.0)
    return {"workload": "cfg2 Gaussian sketch: W 4096x4096 fp32 (config 2) times Omega 4096x48 (fp32-rounded "
                        "N(0,1)), Y fp64", "us_per_call": us,
            "kernels_us": {k: v[0] * 1e3 for k, v in prof.items()},
            "simt_reference_us": 208.0,
            "roofline": {"kernel": "k_sketch_tc", "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOP/s (int8)",
                         "frac": ach / peak, "peak_source": src + " (2 x bf16)", "traffic": None,
                         "ms_per_launch": main_ms},
            "hbm_floor_us": M_ROWS * N_COLS * 4 / (peaks["hbm_gbs"] * 1e9) * 1e6}


def run_cfg5(h, ws, rank, lrank, steps, warmup, peaks, src):
    """Config 5 at full size, row-sharded over the ws ranks (each generates its shard on device)."""
    import torch
    import synth
    from paper_1710_07946_b200 import lra
    m, n = C5_M, C5_N
    rows = m // ws
    row0 = rank * rows
    t0 = time.time()
    U, V = synth.config5_factors(0, m, n)
    Wt = synth.config5_torch(0, m, n, row0=row0, rows=rows, factors=(U, V))
    del U, V
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    mult = synth.multiplier_abridged(0, n, C5_D, C5_K, "arht")
    M = lra.Multiplier(mult)
    W = lra.Dense(Wt, row0=row0, m_global=m if ws > 1 else 0)      # one rank: the unsharded path
    f64 = dict(dtype=torch.float64, device="cuda")
    Y = torch.empty((C5_K, rows), **f64)
    I = torch.empty(C5_K, dtype=torch.int64, device="cuda")
    J = torch.empty(C5_K, dtype=torch.int64, device="cuda")
    Uo = torch.empty((C5_K, C5_K), **f64)
    A = torch.empty((C5_R, rows), **f64)
    B = torch.empty((n, C5_R), **f64)
    num2 = torch.empty(1, **f64)
    den2 = torch.empty(1, **f64)
    stats = lra.new_stats(1, "cuda")

    def step(i):
        lra.lra_preprocess(h, W, M, Y)
        lra.lra_cross_approx(h, W, Y, None, C5_R, C5_K, C5_K, C5_T, I, J, Uo, A, B, stats)
        lra.lra_cur_residual(h, W, A, B, C5_R, num2, den2, prec=lra.LRA_RECON_FAST)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    l0 = h.launches()
    ms = _timed(step, steps, ws, torch.cuda.current_stream()) / steps
    launches = (h.launches() - l0) / steps
    prof, iso_ms = _isolated(h, step, 1, ws)
    st = lra.stats_to_numpy(stats)[0]
    rho = float(np.sqrt(num2.item() / den2.item()))
    sk = sum(v[0] for k, v in prof.items() if k.startswith("k_sketch"))
    rs = sum(v[0] for k, v in prof.items() if k in ("k_split", "k_residual_tc", "k_reduce"))
    rtc = prof.get("k_residual_tc", (0.0, 1))[0]
    sk, rs, rtc = (_max_over_ranks(x, ws) for x in (sk, rs, rtc))
    sk_bytes = m * (1 << C5_D) * _fibers(mult, n, C5_D) * 4 + m * C5_K * 8
    rs_bytes = m * n * 4 + (m * C5_R + C5_R * n) * 8
    out = {"metric": C5_METRIC, "value": 1e3 / ms, "unit": "matrices/s", "ms_per_step": ms, "steps": steps,
           "scaling": "strong", "config": {"workload": C5_WORKLOAD, "rows_per_rank": rows, "gen_s": round(gen_s, 1),
                                           "l2": "inputs_gt_l2 (8.6-68.7 GB per rank)"},
           "isolated_ms_per_step": iso_ms, "kernels_ms": {k: v[0] for k, v in prof.items()},
           "preprocess": _roof("k_sketch (aggregate)", sk_bytes, sk, peaks, src) if sk > 0 else None,
           "residual": _roof("split+k_residual_tc+reduce (aggregate)", rs_bytes, rs, peaks, src) if rs > 0 else None,
           "residual_tc_only": _roof("k_residual_tc (aggregate, W bytes)", m * n * 4, rtc, peaks, src) if rtc > 0 else None,
           "gpu_launches_per_step": launches,
           "status": int(st["status"]), "rho": rho, "lu_steps": int(st["lu_steps"]), "swaps": int(st["swaps"]),
           "cert_rows": float(st["cert_rows"]), "cert_cols": float(st["cert_cols"])}
    for key in ("preprocess", "residual", "residual_tc_only"):
        if out[key] and ws > 1:
            out[key]["per_gpu_frac"] = out[key]["frac"] / ws
    del Wt
    torch.cuda.empty_cache()
    return out


def run_cfg3(h, ws, rank, steps, warmup, peaks, src):
    """Config 3: the 4096 Cauchy blocks dealt out in contiguous ranges, lra_batch per rank."""
    import torch
    import synth
    from paper_1710_07946_b200 import lra, pipeline
    per = C3_NB // ws
    b0 = rank * per
    s, t = synth.cauchy_params(0, C3_NB, C3_M, C3_M)
    Wt = synth.cauchy_blocks_torch(s[b0:b0 + per], t[b0:b0 + per], "cuda")
    mult = synth.multiplier_sparse_batch(0, C3_NB, C3_M, C3_K)
    mb = dict(mult, sp_row=mult["sp_row"][b0:b0 + per], sp_sign=mult["sp_sign"][b0:b0 + per], nb=per)
    M = lra.Multiplier(mb)
    W = lra.Dense(Wt)
    bufs = pipeline.BatchBuffers(per, C3_R, C3_K)

    def step(i):
        pipeline.cur_batch(h, W, M, C3_R, C3_K, C3_T, per, bufs=bufs)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    ms = _timed(step, steps, ws, torch.cuda.current_stream()) / steps
    prof, iso_ms = _isolated(h, step, 1, ws)
    st = lra.stats_to_numpy(bufs.stats)
    rho = np.sqrt(bufs.num2.cpu().numpy() / bufs.den2.cpu().numpy())
    w_bytes = C3_NB * C3_M * C3_M * 4
    out = {"metric": C3_METRIC, "value": C3_NB / (ms / 1e3), "unit": "blocks/s", "ms_per_step": ms,
           "steps": steps, "scaling": "strong (fixed 4096-block batch dealt to ranks)",
           "config": {"workload": C3_WORKLOAD, "blocks_per_rank": per},
           "hbm_frac_of_step": (w_bytes / ws) / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
           "isolated_ms_per_step": iso_ms, "kernels_ms": {k: v[0] for k, v in prof.items()},
           "ok_blocks": int(np.sum(st["status"] == 0)), "median_rho": float(np.median(rho))}
    del Wt
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- headline (config 2)
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=90)
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2, 3, 4],
                    help="batches in flight (S > 1: consecutive steps rotate over S handles and streams)")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg5", "cfg3"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary workloads (cfg5, cfg3)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="few steps, no clocks/e2e/baseline/extras (for ncu)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    if args.warmup < 3 and not args.profile_only:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import synth
    from paper_1710_07946_b200 import Handle, lra, nccl_unique_id, pipeline

    ws, rank, lrank = _dist()
    if ws != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; measuring {ws} rank(s)", file=sys.stderr)
    torch.cuda.set_device(lrank)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    peaks, peaks_src = _peaks()
    # the handle: an NCCL communicator over the ranks for the row-sharded config-5 path
    nid = [None]
    if ws > 1:
        nid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
    h = Handle(lrank, nccl_id=nid[0], nranks=ws, rank=rank)
    st = torch.cuda.current_stream()

    if args.workload != "cfg2":
        fn = run_cfg5 if args.workload == "cfg5" else run_cfg3
        a = (h, ws, rank, lrank) if args.workload == "cfg5" else (h, ws, rank)
        clocks = None if args.profile_only else Clocks(lrank)
        if clocks:
            clocks.ready()
        t0 = time.time()
        res = fn(*a, max(1, args.steps), args.warmup, peaks, peaks_src)
        if clocks:
            clocks.window(t0, time.time())
        if rank == 0:
            res.update({"n_gpus": ws, "warmup": args.warmup, "higher_is_better": True, "vs_baseline": None,
                        "dtype": "f64", "data": "synthetic", "clocks": clocks.stop() if clocks else None,
                        "gpu": torch.cuda.get_device_name(lrank)})
            print(json.dumps(res), flush=True)
        if ws > 1:
            dist.destroy_process_group()
        return

    B = args.batch
    mult = synth.multiplier_abridged(0, N_COLS, DEPTH, K, "arht")
    M = lra.Multiplier(mult)
    host = [_gen_batch([rank * 100000 + p * B + i for i in range(B)]) for p in range(2)]
    pools = [torch.from_numpy(hb).cuda() for hb in host]
    Ws = [lra.Dense(p) for p in pools]
    bufs = pipeline.BatchBuffers(B, R, K)
    # Two batches in flight: consecutive steps alternate between two handles (each with its own
    # side streams and scratch) on two streams, so one batch's tail (the last group's nucleus,
    # factors and residual) overlaps the next batch's C-A waves.  The timed region spans both
    # streams (they wait on the start event; the end event waits on both).
    hs = [h] + [Handle(lrank) for _ in range(args.streams - 1)]
    sts = [torch.cuda.Stream() for _ in hs] if len(hs) > 1 else [st]
    bufsx = [bufs] + [pipeline.BatchBuffers(B, R, K) for _ in hs[1:]]

    def step(i):
        j = i % len(hs)
        pipeline.cur_batch(hs[j], Ws[i % 2], M, R, K, SWEEPS, B, bufs=bufsx[j], stream=sts[j])

    def step1(i):                      # one handle, the current stream (isolation pass)
        pipeline.cur_batch(h, Ws[i % 2], M, R, K, SWEEPS, B, bufs=bufs)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    for bx in bufsx:
        stats = lra.stats_to_numpy(bx.stats)
        assert np.all(stats["status"] == 0), stats
    clocks = None if args.profile_only else Clocks(lrank)
    if clocks:
        clocks.ready()
        step(0)                        # one more untimed step: the GPU back at load clocks after the wait
        torch.cuda.synchronize()
    l0 = sum(x.launches() for x in hs)
    t0 = time.time()
    ms = _timed(step, args.steps, ws, st, sts)
    t1 = time.time()
    if clocks:
        clocks.window(t0, t1)
    launches = sum(x.launches() for x in hs) - l0
    clk = clocks.stop() if clocks else None
    total = ws * B * args.steps
    value = total / (ms / 1e3)
    stats = lra.stats_to_numpy(bufs.stats)
    mean_loops = float(np.mean(stats["loops_done"]))
    pivot_steps = float(np.mean(stats["lu_steps"] + stats["swaps"]))

    # ---- isolation pass: the same two batches, kernels serialized, device time per kernel
    iso_steps = 2
    prof, iso_ms = _isolated(h, step1, iso_steps, ws)
    kern_sum = sum(v[0] for v in prof.values())
    kernels = {k: {"ms_per_step": v[0], "launches_per_step": v[1], "share": v[0] / kern_sum}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    dom = max(prof.items(), key=lambda kv: kv[1][0])[0]

    def per_launch(name):
        ms_step, nl = prof[name]
        return ms_step / nl, B / nl         # ms per launch, matrices per launch

    stage = {}
    for name in prof:
        if name.startswith("k_sketch"):
            ml, mats = per_launch(name)
            stage["preprocess"] = _roof(name, alg_bytes_cfg2(name, mult, mats), ml, peaks, peaks_src)
        if name == "k_residual_tc":
            ml, mats = per_launch(name)
            stage["residual_tc"] = _roof(name, alg_bytes_cfg2(name, mult, mats), ml, peaks, peaks_src)
            tr = _ncu_traffic(name, mats)
            if tr:
                stage["residual_tc"]["traffic"] = tr["bytes_per_launch"]
                stage["residual_tc"]["traffic_source"] = tr["source"]
    rs_ms = sum(prof[k][0] for k in ("k_split", "k_residual_tc", "k_reduce") if k in prof)
    if rs_ms > 0:
        stage["residual_stage"] = _roof("k_split+k_residual_tc+k_reduce", alg_bytes_cfg2("residual_stage", mult, B),
                                        rs_ms, peaks, peaks_src)
    ml, mats = per_launch(dom)
    if dom in ("k_ca",):
        roof = _roof(dom, alg_bytes_cfg2(dom, mult, mats, loops=mean_loops), ml, peaks, peaks_src)
        roof["note"] = ("latency-bound pivot chain (DESIGN.md §6.1): algorithmic gather bytes over the isolated "
                        "launch time; 'latency' gives the per-pivot-step cost")
        roof["latency"] = {"launch_ms": ml, "matrices_per_launch": mats, "pivot_steps_per_matrix": pivot_steps,
                           "us_per_pivot_step": ml * 1e3 / max(1.0, pivot_steps)}
    else:
        roof = dict(stage.get("residual_tc" if dom == "k_residual_tc" else "preprocess")
                    or _roof(dom, 0, ml, peaks, peaks_src))
    tr = _ncu_traffic(dom, mats)
    if tr and roof.get("traffic") is None:
        roof["traffic"] = tr["bytes_per_launch"]
        roof["traffic_source"] = tr["source"]

    # ---- e2e through the public API with host buffers: H2D of each batch overlapped with the
    # previous batch's compute (copy stream + events), D2H of the per-matrix results
    e2e = None
    if not args.no_e2e and not args.profile_only:
        pin = [torch.from_numpy(hb).pin_memory() for hb in host]
        dev = [torch.empty_like(pools[0]) for _ in range(2)]
        Wd = [lra.Dense(d) for d in dev]
        outs = [[torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (bufs.I, bufs.J, bufs.U, bufs.num2,
                                                                           bufs.den2)] for _ in range(2)]
        cs = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        ke = max(4, min(args.steps, 12))

        def e2e_run(nsteps):
            with torch.cuda.stream(cs):
                dev[0].copy_(pin[0], non_blocking=True)
                copied[0].record(cs)
            for i in range(nsteps):
                if i + 1 < nsteps:          # prefetch the next batch while this one computes
                    with torch.cuda.stream(cs):
                        if i >= 1:
                            cs.wait_event(used[(i + 1) % 2])
                        dev[(i + 1) % 2].copy_(pin[(i + 1) % 2], non_blocking=True)
                        copied[(i + 1) % 2].record(cs)
                st.wait_event(copied[i % 2])
                pipeline.cur_batch(h, Wd[i % 2], M, R, K, SWEEPS, B, bufs=bufs)
                used[i % 2].record(st)
                for o, x in zip(outs[i % 2], (bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2)):
                    o.copy_(x, non_blocking=True)

        e2e_run(2)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(st)
        e2e_run(ke)
        f1.record(st)
        torch.cuda.synchronize()
        ems = _max_over_ranks(f0.elapsed_time(f1), ws)
        d2h = sum(x.numel() * x.element_size() for x in (bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2))
        h2d = int(pools[0].numel() * 4)
        # the host link's own rate: the same pinned batch copied alone, back to back (best of 3)
        link = 0.0
        for _ in range(3):
            l0 = torch.cuda.Event(enable_timing=True)
            l1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                l0.record(cs)
                dev[0].copy_(pin[0], non_blocking=True)
                l1.record(cs)
            torch.cuda.synchronize()
            link = max(link, h2d / (l0.elapsed_time(l1) / 1e3) / 1e9)
        h2d_gbs = h2d * ke / (ems / 1e3) / 1e9
        e2e = {"value": ws * B * ke / (ems / 1e3), "unit": "matrices/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h), "h2d_GBs_per_gpu": h2d_gbs,
               "h2d_link_GBs": link, "pcie_frac": h2d_gbs / link if link > 0 else None,
               "note": "H2D of batch i+1 overlaps batch i's compute; pcie_frac = the step's H2D rate over the "
                       "link rate measured alone (a pinned copy of the same batch): near 1 = PCIe-bound"}
        del dev, Wd, pin

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile_only:
        cpu = cpu_baseline()

    # ---- secondary workloads (config 5 row-sharded, config 3 dealt), device-timed
    extra = {}
    if not args.no_extra and not args.profile_only:
        del pools, Ws
        torch.cuda.empty_cache()
        if rank == 0:
            try:
                extra["sketch_gaussian_tc"] = run_sketch_tc(h, peaks, peaks_src)
            except Exception as ex:
                extra["sketch_gaussian_tc"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        for name, fn, a in (("cfg3", run_cfg3, (h, ws, rank)), ("cfg5", run_cfg5, (h, ws, rank, lrank))):
            try:
                extra[name] = fn(*a, 5 if name == "cfg5" else 10, 2 if name == "cfg5" else 3, peaks, peaks_src)
            except Exception as ex:          # report, keep the headline
                extra[name] = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "matrices/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "batch_per_gpu": B, "l2": "inputs_gt_l2 (2 alternating batches of "
                           f"{B} x 67 MB per GPU)", "parallelism": f"dp{ws} (independent matrices per rank)",
                           "batches_in_flight": len(hs)},
                "roofline": roof, "stage_rooflines": stage,
                "isolation": {"ms_per_step": iso_ms, "kernel_ms_sum": kern_sum, "steps": iso_steps,
                              "note": "same batches, lra_batch groups serialized on one stream, event pair per "
                                      "kernel on its launch stream (device time, no queueing)"},
                "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "workloads": extra, "gpu": torch.cuda.get_device_name(lrank)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
