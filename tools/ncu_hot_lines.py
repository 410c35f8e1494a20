"""Aggregate ncu warp-stall samples per CUDA source line (cuda,sass view) of one kernel.
usage: python tools/ncu_hot_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None
lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 6 and r[0].isdigit():
        try:
            lines.append((float(r[4] or 0), f"{fname}:{r[0]}", r[1].strip()))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
for s, loc, src in sorted(lines, key=lambda x: -x[0])[:n]:
    print(f"{s / tot * 100:5.1f}%  {loc:16s} {src[:100]}")
