timeout 600 python -m pytest tests/test_edges.py -m gpu -q > gpurun_out/r2c50_edges.log 2>&1; echo "rc=$?" >> gpurun_out/r2c50_edges.log
timeout 120 tools/microbench/dmma_issue > gpurun_out/r2c50_dmma_issue.txt 2>&1
