#!/bin/bash
# headline bench under diagnostic settings: "NAME ENV..." per line in $CASES (separated by ';')
mkdir -p gpurun_out
: > gpurun_out/bench_var.txt
IFS=';' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  name=${c%% *}; envs=${c#* }; [ "$envs" = "$name" ] && envs=""
  env $envs timeout 300 python bench.py --steps 30 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/bv_$name.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/bv_$name.json')); print('$name', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/bench_var.txt
done
