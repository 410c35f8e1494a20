#!/bin/bash
mkdir -p gpurun_out
A="${RES_ARGS:-16384 16384 32 1}"
timeout 120 python tools/resid_bench.py $A > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resid -s 5 -c 1 -f -o gpurun_out/resid_prof python tools/resid_bench.py $A > gpurun_out/ncu1.log 2>&1; echo "ncu=$?"
