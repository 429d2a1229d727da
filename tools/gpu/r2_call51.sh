timeout 120 tools/microbench/dmma_issue > gpurun_out/r2c51_dmma_issue.txt 2>&1
