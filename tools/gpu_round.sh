#!/bin/bash
# One gpurun call: smoke, GPU tests, bench line, launch list, ncu --set full of the hot kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/host.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_EXTRA} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
cat gpurun_out/bench.json | head -c 3000
if [ -z "$NO_NCU" ]; then
P="python bench.py --profile-only --steps 1 --warmup 1 --batch 14"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K:-k_cacl|k_residual_tc|k_sketch|k_nucleus|k_split}" -s ${NCU_S:-0} -c ${NCU_C:-5} -f -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
fi
