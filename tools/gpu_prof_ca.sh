#!/bin/bash
# tests, then ncu --set full of the C-A and nucleus kernels on one config-2 matrix
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 120 python tools/ca_phases.py arht > gpurun_out/phases.json 2>&1 && python -c "import json;d=json.load(open('gpurun_out/phases.json'));print({k:round(v,1) for k,v in d['phases_us'].items() if v}, {k:round(v[0]*1e3,1) for k,v in d['kernels_ms'].items()})" && \
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_cacl|k_nucleus" -c 2 -f -o gpurun_out/prof_ca python tools/ca_phases.py arht > gpurun_out/ncu_ca.log 2>&1; echo "ncu=$?"
