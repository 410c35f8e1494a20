#!/bin/bash
# ncu --set full capture of k_sketch_tc (config 2 Gaussian sketch) through lra_preprocess
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sketch_tc -s 1 -c 1 \
  -o gpurun_out/stc_full -f python tools/sketch_tc_time.py 3 > gpurun_out/stc_ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/stc_ncu.log
