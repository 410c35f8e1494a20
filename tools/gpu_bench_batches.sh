#!/bin/bash
# headline bench at several batch sizes (two batches in flight)
mkdir -p gpurun_out
: > gpurun_out/bench_batches.txt
for B in ${BATCHES:-60 90 120 150}; do
  timeout 300 python bench.py --batch $B --steps 30 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/bb_$B.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bb_$B.json')); print($B, round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/bench_batches.txt
done
