#!/bin/bash
# residual parity tests + timings across shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "residual or config2_full or config3_batch or config1 or fast or ragged or bench_configuration or config5" > gpurun_out/pytest_resid.log 2>&1; echo "pytest=$?" >> gpurun_out/pytest_resid.log
for args in "16384 16384 32 0" "32768 32768 64 0" "32768 32768 32 0" "65536 32768 64 0" "16384 16384 32 1" "4096 4096 32 1"; do
  timeout 120 python tools/resid_bench.py $args 2>&1 | tail -1
done > gpurun_out/resid_bench.txt
