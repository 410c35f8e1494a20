#!/bin/bash
# residual timings: default build vs the diagnostic variants named in $VARS (liblra_<v>.so)
mkdir -p gpurun_out
: > gpurun_out/resid_var.txt
for v in base $VARS; do
  so=paper_1710_07946_b200/liblra.so; [ "$v" != base ] && so=paper_1710_07946_b200/liblra_$v.so
  for args in "32768 32768 64 0" "32768 32768 32 0" "16384 16384 32 1" "4096 4096 32 1"; do
    echo -n "$v: " >> gpurun_out/resid_var.txt
    LRA_SO=$so timeout 120 python tools/resid_bench.py $args 2>&1 | tail -1 >> gpurun_out/resid_var.txt
  done
done
