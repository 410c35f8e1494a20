#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/resid_prof.txt
for args in "32768 32768 64 0" "32768 32768 32 0" "16384 16384 32 1"; do
  LRA_SO=paper_1710_07946_b200/liblra_prof.so timeout 120 python tools/resid_bench.py $args 2>&1 | tail -2 >> gpurun_out/resid_prof.txt
done
