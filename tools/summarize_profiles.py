"""Summaries of a gpu_round.sh call for profiles/: the ncu launch list (per-kernel share of
the step, cold-cache and serialised) and the key metrics of the ncu --set full capture.
usage: python tools/summarize_profiles.py OUTDIR TAG"""
import collections
import csv
import os
import subprocess
import sys

out_dir, tag = sys.argv[1], sys.argv[2]
rep = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/prof.ncu-rep"
launches = sys.argv[4] if len(sys.argv) > 4 else "gpurun_out/launches.csv"
os.makedirs(out_dir, exist_ok=True)
rows = list(csv.reader(open(launches))) if os.path.exists(launches) else []
hdr = None
d = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        d[x["Kernel Name"][:80]].append(float(x["Metric Value"]))
tot = sum(sum(v) for v in d.values()) or 1.0
with open(os.path.join(out_dir, f"launches_{tag}.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --profile-only "
            "--steps 1 --warmup 1 --batch 14\n(cold-cache, serialised launches: compare shares, not absolutes)\n")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"{k:80s} n={len(v):4d} total={sum(v)/1e3:10.1f}us share={sum(v)/tot:.3f} avg={sum(v)/len(v)/1e3:9.1f}us\n")
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__cluster_dim_x"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u = r[0], r[1]
idx = [h.index(w) for w in want if w in h]
with open(os.path.join(out_dir, f"ncu_full_{tag}.txt"), "w") as f:
    f.write(f"ncu --set full --clock-control none --import-source on ({os.path.basename(rep)})\n")
    for row in r[2:]:
        f.write("; ".join(f"{h[i]}={row[i]} {u[i]}".strip() for i in idx) + "\n")
print(open(os.path.join(out_dir, f"launches_{tag}.txt")).read()[:3000])
# the hottest source lines (stall samples) of every captured kernel, for the committed summary
try:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    with open(os.path.join(out_dir, f"ncu_hot_{tag}.txt"), "w") as f:
        kern, hdr2 = None, None
        rows2 = []
        for row in csv.reader(src.splitlines()):
            if len(row) >= 2 and row[0] == "Kernel Name":
                kern = row[1]
                continue
            if row and row[0] == "Address":
                hdr2 = row
                continue
            if hdr2 and kern and len(row) == len(hdr2):
                rows2.append((kern, dict(zip(hdr2, row))))
        by = collections.defaultdict(list)
        for k, x in rows2:
            by[k].append(x)
        for k, xs in by.items():
            tot2 = sum(float(x.get("Warp Stall Sampling (All Samples)") or 0) for x in xs) or 1.0
            f.write(f"== {k[:120]}  (stall samples {tot2:.0f})\n")
            for x in sorted(xs, key=lambda x: -float(x.get("Warp Stall Sampling (All Samples)") or 0))[:12]:
                f.write(f"  {float(x.get('Warp Stall Sampling (All Samples)') or 0) / tot2 * 100:5.1f}%  "
                        f"{x.get('Source', '')[:100]}  executed={x.get('Instructions Executed', '')}\n")
except Exception as ex:  # the summary is best effort
    print("source page:", ex)
