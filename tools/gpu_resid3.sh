#!/bin/bash
# residual timings across shapes + one ncu --set full capture of the config-5-shaped FAST kernel
mkdir -p gpurun_out
for args in "16384 16384 32 0" "32768 32768 64 0" "32768 32768 32 0" "65536 32768 64 0" "16384 16384 32 1" "4096 4096 32 1"; do
  timeout 120 python tools/resid_bench.py $args 2>&1 | tail -1
done > gpurun_out/resid_bench.txt
A="32768 32768 64 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resid -s 5 -c 1 -f -o gpurun_out/resid_r64 python tools/resid_bench.py $A > gpurun_out/ncu_r64.log 2>&1; echo "ncu=$?"
