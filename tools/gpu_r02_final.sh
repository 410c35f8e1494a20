#!/bin/bash
# Round-2 closing evidence: smoke, GPU tests, bench line, ncu launch list of the bench's profile pass.
mkdir -p gpurun_out/summ
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
P="python bench.py --profile-only --steps 1 --warmup 1 --batch 14"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
du -sh gpurun_out
