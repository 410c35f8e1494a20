#!/bin/bash
# C-A iteration: regressions vs the recorded fingerprint, GPU tests, phases, bench.
mkdir -p gpurun_out
timeout 300 python tools/ca_regress.py gpurun_out/ca_regress_new.json > gpurun_out/regress_new.log 2>&1; echo "regress=$?"
python tools/ca_compare.py tools/ca_regress_baseline.json gpurun_out/ca_regress_new.json
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 120 python tools/ca_phases.py arht > gpurun_out/phases.json 2>&1; head -14 gpurun_out/phases.json
timeout 600 python bench.py --no-cpu-baseline ${BENCH_EXTRA} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"; head -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
