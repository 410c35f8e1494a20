#!/bin/bash
# tests + kernel phases + bench at several batch-group counts
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 120 python tools/ca_phases.py arht > gpurun_out/phases.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/phases.json'));print({k:round(v,1) for k,v in d['phases_us'].items() if v}, {k:round(v[0]*1e3,1) for k,v in d['kernels_ms'].items()})"
for g in ${GROUPS_LIST:-2 4 8}; do LRA_BATCH_GROUPS=$g timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_g$g.json 2>&1; echo "groups=$g"; python -c "import json;d=json.load(open('gpurun_out/bench_g$g.json'));print(round(d['value']), round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"; done
