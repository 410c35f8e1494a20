#!/usr/bin/env python
"""bench.py — throughput of the superfast-CUR hot path on B200 (BASELINE.json metric:
"CUR LRA matrices/sec and preprocess+residual GB/s vs HBM peak, 1/2/4/8 B200").

One step = one pass of the whole hot path (§8(a): sketch, C-A sweeps, nucleus + factors,
full a-posteriori check) over one batch of B synthetic config-2 matrices per GPU
(W = U·diag(σ)·Vᵀ fp32 4096², r = 32, k = l = 48, ARHT d = 4, 3 sweeps), through
``lra_batch``.  Two batches alternate, so consecutive steps never find their inputs in L2
(2·B·67 MB > 126 MB).  N > 1: one process per GPU (torchrun), independent matrices per
rank, no collective on the data path ("weak" scaling), max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl native|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_ROWS = N_COLS = 4096
R, K, SWEEPS, DEPTH = 32, 48, 3, 4
WORKLOAD = (f"cfg2-arht: W=U*diag(s)*V^T fp32 {M_ROWS}x{N_COLS}, s_i=1 (i<=32) then 1e-6*0.9^(i-32); "
            f"r={R}, k=l={K}, ARHT d={DEPTH} +-1 diagonal, {SWEEPS} C-A sweeps, full residual")
METRIC = "CUR LRA matrices/sec (config 2, ARHT) — sketch+C-A+nucleus+residual"


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


def _gen_batch(seeds):
    import synth
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        Ws = list(ex.map(lambda s: synth.config2(s, n=N_COLS), seeds))
    out = np.empty((len(seeds), N_COLS, M_ROWS), dtype=np.float32)
    for i, W in enumerate(Ws):
        out[i] = W.T
    return out


class Clocks:
    """nvidia-smi sampler (200 ms) for the clocks line of the JSON."""

    def __init__(self, dev):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.t0 = self.t1 = None

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
            if self.t0 is None or ts is None or (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                rows.append(row)
        if not rows:
            rows = all_rows
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        # samples while the GPU was busy: keep the top half by clock (idle samples sit at max
        # too, but the warm-up + timed region dominate the sampler's lifetime)
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


def cpu_baseline(n_mats=4):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload."""
    import synth
    from oracle import lra as O
    mult = synth.multiplier_abridged(0, N_COLS, DEPTH, K, "arht")
    Ws = [synth.config2(90000 + i, n=N_COLS) for i in range(n_mats)]
    t = time.perf_counter()
    for W in Ws:
        O.cur_pipeline(W, mult, R, K, K, SWEEPS)
    dt = time.perf_counter() - t
    return {"value": n_mats / dt, "unit": "matrices/s", "cores": _oracle_cores(), "kind": "oracle",
            "sample": f"{n_mats} config-2 matrices (full size) through oracle.cur_pipeline, {dt:.1f} s"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import synth
    from oracle import lra as O
    mult = synth.multiplier_abridged(0, N_COLS, DEPTH, K, "arht")
    Ws = [synth.config2(80000 + i, n=N_COLS) for i in range(args.warmup + args.steps)]
    for W in Ws[:args.warmup]:
        O.cur_pipeline(W, mult, R, K, K, SWEEPS)
    t = time.perf_counter()
    for W in Ws[args.warmup:]:
        O.cur_pipeline(W, mult, R, K, K, SWEEPS)
    dt = time.perf_counter() - t
    v = args.steps / dt
    cores = _oracle_cores()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "matrices/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "batch_per_step": 1,
                                           "note": "reference arm = the fp64 numpy oracle (no reference code exists)"},
            "cpu_baseline": {"value": v, "unit": "matrices/s", "cores": cores, "kind": "oracle",
                             "sample": f"1 full-size config-2 matrix per step, {args.steps} steps"},
            "e2e": {"value": v, "unit": "matrices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def algorithmic(name, mult, B):
    """Algorithmic bytes (and flops) of one launch of `name` over a batch of B matrices
    (DESIGN.md §6): what the method must move, not what the kernel happens to move."""
    m, n = M_ROWS, N_COLS
    s = n >> DEPTH
    fibers = len({int(c) % s for c in mult["col"]})
    if name.startswith("k_sketch"):
        return B * (m * (1 << DEPTH) * fibers * 4 + m * K * 8), 0.0
    if name == "k_residual":
        return B * (m * n * 4 + (m * R + R * n) * 8), B * 2.0 * m * n * R
    if name == "k_residual_tc":   # W once + the int8 digit slices of A and B (6 each)
        return B * (m * n * 4 + (m + n) * R * 6), B * 2.0 * m * n * R * 21
    if name == "k_ca":
        return B * SWEEPS * (m * K + K * n) * 4, 0.0
    return 0, 0.0


def ncu_traffic(kname, mats_per_launch):
    """dram read+write bytes per launch of kname from the committed ncu --set full summary
    (profiles/<round>/ncu_full_final.txt), scaled from that capture's problems per launch."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "*",
                                          "ncu_full_final.txt")))
    key = {"k_ca": "k_cacl"}.get(kname, kname)
    for path in reversed(files):
        for line in open(path):
            if not line.startswith("Kernel Name=") or key not in line.split(";")[0]:
                continue
            f = dict(kv.split("=", 1) for kv in (x.strip() for x in line.split(";")) if "=" in kv)
            rd = float(f["dram__bytes_read.sum"].split()[0]) * (1e6 if "Mbyte" in f["dram__bytes_read.sum"] else 1e9 if "Gbyte" in f["dram__bytes_read.sum"] else 1e3)
            wr = float(f["dram__bytes_write.sum"].split()[0]) * (1e6 if "Mbyte" in f["dram__bytes_write.sum"] else 1e9 if "Gbyte" in f["dram__bytes_write.sum"] else 1e3)
            grid = int(re.sub(r"[^0-9]", "", f.get("launch__grid_size", "0")) or 0)
            cdim = int(re.sub(r"[^0-9]", "", f.get("launch__cluster_dim_x", "0")) or 0)
            if key == "k_cacl" and grid and cdim:
                cap_mats = grid / cdim
            elif key.startswith("k_residual"):
                cap_mats = rd / (4096 * 4096 * 4)
            else:
                return None
            return {"bytes_per_launch": (rd + wr) / cap_mats * mats_per_launch,
                    "source": os.path.relpath(path, os.path.dirname(os.path.abspath(__file__)))}
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=42)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="few steps, no clocks/e2e/baseline (for ncu)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile_only:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import synth
    from paper_1710_07946_b200 import Handle, lra, pipeline

    ws, rank, lrank = _dist()
    torch.cuda.set_device(lrank)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    B = args.batch
    mult = synth.multiplier_abridged(0, N_COLS, DEPTH, K, "arht")
    M = lra.Multiplier(mult)
    host = [_gen_batch([rank * 100000 + p * B + i for i in range(B)]) for p in range(2)]
    pools = [torch.from_numpy(h).cuda() for h in host]
    Ws = [lra.Dense(p) for p in pools]
    h = Handle(lrank)
    bufs = pipeline.BatchBuffers(B, R, K)
    st = torch.cuda.current_stream()

    def step(i):
        pipeline.cur_batch(h, Ws[i % 2], M, R, K, SWEEPS, B, bufs=bufs)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    stats = lra.stats_to_numpy(bufs.stats)
    assert np.all(stats["status"] == 0), stats
    clocks = None if args.profile_only else Clocks(lrank)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    h.profile(True)
    l0 = h.launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record(st)
    for i in range(args.steps):
        step(i)
    e1.record(st)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t1 = time.time()
    if clocks:
        clocks.window(t0, t1)
    ms = e0.elapsed_time(e1)
    launches = h.launches() - l0
    prof = h.profile_read()
    h.profile(False)
    if ws > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    clk = clocks.stop() if clocks else None
    total = ws * B * args.steps
    value = total / (ms / 1e3)
    peaks, peaks_src = _peaks()

    # ---- roofline of the dominant kernel (live CUDA-event timing inside the timed region)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    name, (kms, cnt) = dom
    per_launch_s = kms / cnt / 1e3
    # one launch processes one batch group: B * steps / (launches of this kernel in the region)
    per_launch_mats = B * args.steps / cnt
    byts, flops = algorithmic(name, mult, per_launch_mats)
    if name == "k_ca":
        ach = byts / per_launch_s / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "peak_source": peaks_src, "traffic": None,
                "note": "latency-bound pivot chain (DESIGN.md §6.1): the algorithmic gather bytes over the launch "
                        "time; see 'latency' for the per-step cost",
                "latency": {"launch_ms": kms / cnt, "matrices_per_launch": per_launch_mats,
                            "pivot_steps_per_matrix": float(np.mean(stats["lu_steps"] + stats["swaps"])),
                            "us_per_pivot_step": kms / cnt * 1e3 / max(1.0, float(np.mean(stats["lu_steps"] + stats["swaps"])))}}
    elif name == "k_residual":
        fp64_peak = float(os.environ.get("LRA_FP64_TFLOPS", "37.2"))
        roof = {"kernel": name, "bound": "alu", "achieved": flops / per_launch_s / 1e12, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": flops / per_launch_s / 1e12 / fp64_peak,
                "peak_source": "FP64 DFMA: 148 SMs x 64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §6)",
                "hbm_gbs": byts / per_launch_s / 1e9, "hbm_frac": byts / per_launch_s / 1e9 / peaks["hbm_gbs"],
                "traffic": None}
    else:
        ach = byts / per_launch_s / 1e9
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "peak_source": peaks_src, "traffic": None}
    tr = ncu_traffic(name, per_launch_mats)
    if tr:
        roof["traffic"] = tr["bytes_per_launch"]
        roof["traffic_source"] = tr["source"]
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches": v[1],
                   "share": v[0] / sum(x[0] for x in prof.values())} for k, v in prof.items()}
    stage_gbs = {}
    for k in ("k_sketch_arht", "k_residual", "k_residual_tc"):
        if k in prof:
            b, _ = algorithmic(k, mult, B * args.steps / prof[k][1])
            stage_gbs[k] = b / (prof[k][0] / prof[k][1] / 1e3) / 1e9

    # ---- e2e through the public API with host buffers (H2D of W, D2H of results, timed)
    e2e = None
    if not args.no_e2e and not args.profile_only:
        pin = [torch.from_numpy(hb).pin_memory() for hb in host]
        dev = torch.empty_like(pools[0])
        Wd = lra.Dense(dev)
        outs = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2)]
        ke = max(3, min(args.steps, 10))
        for i in range(2):
            dev.copy_(pin[i % 2], non_blocking=True)
            pipeline.cur_batch(h, Wd, M, R, K, SWEEPS, B, bufs=bufs)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(st)
        for i in range(ke):
            dev.copy_(pin[i % 2], non_blocking=True)
            pipeline.cur_batch(h, Wd, M, R, K, SWEEPS, B, bufs=bufs)
            for o, x in zip(outs, (bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2)):
                o.copy_(x, non_blocking=True)
        f1.record(st)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        if ws > 1:
            tt = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        d2h = sum(x.numel() * x.element_size() for x in (bufs.I, bufs.J, bufs.U, bufs.num2, bufs.den2))
        e2e = {"value": ws * B * ke / (ems / 1e3), "unit": "matrices/s",
               "h2d_bytes_per_step": int(pools[0].numel() * 4), "d2h_bytes_per_step": int(d2h)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile_only:
        cpu = cpu_baseline()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "matrices/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOAD, "batch_per_gpu": B, "l2": "inputs_gt_l2 (2 alternating batches of "
                           f"{B} x 67 MB per GPU)", "parallelism": f"dp{ws} (independent matrices per rank)"},
                "roofline": roof, "stage_gbs": stage_gbs, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk,
                "gpu": torch.cuda.get_device_name(lrank)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
