#!/bin/bash
# ncu --set full of the small C-A tier on a config-3 batch (148 blocks), summarized on the box
mkdir -p gpurun_out/summ
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cas -c 1 -o gpurun_out/cas -f \
  env LRA_BATCH_GROUPS=1 python tools/ca_phases_cfg3.py 148 > gpurun_out/cas_ncu.log 2>&1; echo "ncu=$?"
python tools/summarize_profiles.py gpurun_out/summ cas gpurun_out/cas.ncu-rep /nonexistent > /dev/null 2>&1; echo "summ=$?"
rm -f gpurun_out/cas.ncu-rep
