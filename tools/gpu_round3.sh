#!/bin/bash
# Round evidence in one gpurun call: smoke, GPU tests, bench line, ncu launch list and --set full
# summaries of the bench's hot kernels and of the config-5-shaped FAST residual.
mkdir -p gpurun_out/summ
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
P="python bench.py --profile-only --steps 1 --warmup 1 --batch 14"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_cacl|k_resid|k_sketch|k_nucleus|k_split" -s 0 -c 5 -f -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
python tools/summarize_profiles.py gpurun_out/summ final gpurun_out/prof.ncu-rep gpurun_out/launches.csv > /dev/null 2>&1; echo "summ=$?"
R="python tools/resid_bench.py 32768 32768 64 0"
timeout 300 $R > gpurun_out/resid_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_resid -s 5 -c 1 -f -o gpurun_out/resid_full $R > gpurun_out/ncu_resid.log 2>&1; echo "ncu_resid=$?"
python tools/summarize_profiles.py gpurun_out/summ resid_fast_r64 gpurun_out/resid_full.ncu-rep /nonexistent > /dev/null 2>&1
rm -f gpurun_out/prof.ncu-rep
du -sh gpurun_out
