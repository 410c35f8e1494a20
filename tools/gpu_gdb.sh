#!/bin/bash
mkdir -p gpurun_out
export REPS=${REPS:-80} SYNC_EACH=1
timeout 900 /usr/local/cuda/bin/cuda-gdb -q -batch -ex "set cuda break_on_launch none" -ex "run" -ex "info cuda kernels" -ex "bt 8" -ex "x/4i \$pc" -ex "info cuda threads" --args python tools/cfg3_check.py 148 > gpurun_out/gdb.log 2>&1
echo "gdb=$?"
grep -v "^\[New Thread\|^\[Thread\|^\[Detaching\|^rep " gpurun_out/gdb.log | tail -60
