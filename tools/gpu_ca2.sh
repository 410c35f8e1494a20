#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "config2 or config1 or tie or ragged or random_start or batch or qgauss or leverage or rectangular or projective" > gpurun_out/pytest_ca2.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_ca2.log
for sl in 1 2; do LRA_CA_SLOTS=$sl timeout 120 python tools/ca_phases.py arht 2>&1 | python -c "import sys,json; d=json.load(sys.stdin); print('slots', $sl, 'k_ca ms', d['kernels_ms']['k_ca'], {k: round(v,1) for k,v in d['phases_us'].items() if k in ('load','cold_lu','gauss_jordan','product','swap_loop','kernel')})"; done
for sl in 1 2; do LRA_CA_SLOTS=$sl timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extra 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print('slots', $sl, 'bench', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'iso k_ca', round(d['kernels']['k_ca']['ms_per_step'],3))"; done
