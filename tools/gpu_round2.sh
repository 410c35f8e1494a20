#!/bin/bash
# One gpurun call for the round's evidence, everything small written to gpurun_out/ (the .ncu-rep
# files are summarized on the box and removed: gpurun copies back at most 64 MiB).
mkdir -p gpurun_out/summ
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
for B in ${BATCHES:-84 126}; do
  timeout 600 python bench.py --batch $B --steps 30 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/bench_b$B.json 2>/dev/null; echo "bench_b$B=$?"
done
P="python bench.py --profile-only --steps 1 --warmup 1 --batch 14"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_cacl|k_resid|k_sketch|k_nucleus|k_split" -s 0 -c 5 -f -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
python tools/summarize_profiles.py gpurun_out/summ final gpurun_out/prof.ncu-rep gpurun_out/launches.csv > /dev/null 2>&1; echo "summ=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sketch_tc -s 1 -c 1 \
  -o gpurun_out/stc_full -f python tools/sketch_tc_time.py 3 > gpurun_out/stc_ncu.log 2>&1; echo "ncu_stc=$?"
python tools/summarize_profiles.py gpurun_out/summ sketch_tc gpurun_out/stc_full.ncu-rep /nonexistent > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stc.csv python tools/sketch_tc_time.py 3 > /dev/null 2>&1
rm -f gpurun_out/prof.ncu-rep
du -sh gpurun_out
