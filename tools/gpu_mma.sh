#!/bin/bash
mkdir -p gpurun_out
timeout 60 ./tools/mma_issue_bench > gpurun_out/mma_issue.txt 2>&1; cat gpurun_out/mma_issue.txt
