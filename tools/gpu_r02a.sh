#!/bin/bash
# Round-2 check: smoke, GPU tests, bench line (headline + isolation + cfg3/cfg5), TMEM ld microbench.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 120 ./tools/tmem_ld_bench > gpurun_out/tmem_ld.txt 2>&1; echo "tmem=$?"
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
timeout 1800 python -m pytest tests -m gpu -x -q ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
