#!/bin/bash
# config-3 arm under diagnostic settings: "NAME ENV..." per case in $CASES (';'-separated)
mkdir -p gpurun_out
: > gpurun_out/cfg3_var.txt
IFS=';' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  name=${c%% *}; envs=${c#* }; [ "$envs" = "$name" ] && envs=""
  env $envs timeout 300 python bench.py --workload cfg3 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/c3_$name.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c3_$name.json')); print('$name', round(d['value'],1), round(d['ms_per_step'],3))" >> gpurun_out/cfg3_var.txt
done
