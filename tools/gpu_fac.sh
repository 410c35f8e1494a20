#!/bin/bash
# Factor kernels A/B: bit identity against the previous build (LRA_SO), GPU tests, bench line.
mkdir -p gpurun_out
LRA_SO=paper_1710_07946_b200/liblra_prev.so timeout 300 python tools/nuc_compare.py gpurun_out/prev.npz > gpurun_out/fac_prev.log 2>&1; echo "prev=$?"
timeout 300 python tools/nuc_compare.py gpurun_out/new.npz > gpurun_out/fac_new.log 2>&1; echo "new=$?"
python tools/nuc_compare.py --cmp gpurun_out/prev.npz gpurun_out/new.npz > gpurun_out/fac_cmp.log 2>&1; echo "cmp=$?"
rm -f gpurun_out/prev.npz gpurun_out/new.npz
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
