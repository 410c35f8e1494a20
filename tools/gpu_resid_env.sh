#!/bin/bash
# residual timings under diagnostic environment settings: "NAME ENV..." per case in $CASES
mkdir -p gpurun_out
: > gpurun_out/resid_env.txt
IFS=';' read -ra cs <<< "$CASES"
for c in "${cs[@]}"; do
  name=${c%% *}; envs=${c#* }; [ "$envs" = "$name" ] && envs=""
  for args in "32768 32768 64 0" "16384 16384 32 1"; do
    echo -n "$name: " >> gpurun_out/resid_env.txt
    env $envs timeout 120 python tools/resid_bench.py $args 2>&1 | tail -1 >> gpurun_out/resid_env.txt
  done
done
