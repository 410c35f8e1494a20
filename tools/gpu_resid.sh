#!/bin/bash
# residual kernel: parity tests + timings + role counters
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "residual or config2_full or config3_batch or config1 or fast or ragged or bench_configuration" > gpurun_out/pytest_resid.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_resid.log
for args in "16384 16384 32 1" "16384 16384 32 0" "32768 32768 64 0" "32768 32768 64 1" "4096 4096 32 1"; do
  timeout 120 python tools/resid_bench.py $args 2>&1 | tail -1
  LRA_SO=paper_1710_07946_b200/liblra_prof.so timeout 120 python tools/resid_bench.py $args 2>&1 | tail -2 | head -1
done > gpurun_out/resid_bench.txt
cat gpurun_out/resid_bench.txt
