#!/bin/bash
# C-A change check: fingerprints vs the committed baseline, per-phase counters (batch of 15), bench
mkdir -p gpurun_out
timeout 600 python tools/ca_regress.py gpurun_out/fp_new.json > gpurun_out/regress.log 2>&1
python -c "
import json; a=json.load(open('tools/ca_regress_baseline.json')); b=json.load(open('gpurun_out/fp_new.json')); print('fingerprints equal:', a==b, len(a), len(b))" > gpurun_out/fpcmp.txt 2>&1
LRA_BATCH_GROUPS=1 timeout 300 python tools/ca_phases_batch.py 15 > gpurun_out/phases15.json 2>&1
CASES="${CASES:-cur}" bash tools/gpu_bench_var.sh
