#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --workload cfg3 --steps 5 2>&1 | grep -v "^frame" | tail -2 | cut -c1-300; echo "cfg3 alone=$?"
timeout 300 python bench.py --workload cfg5 --steps 3 2>&1 | grep -v "^frame" | tail -2 | cut -c1-300; echo "cfg5 alone=$?"
timeout 600 python bench.py --steps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -v "^frame" | tail -3 | cut -c1-400; echo "no-e2e=$?"
