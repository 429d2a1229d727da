timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -q -k bench_workload > gpurun_out/r2c65_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2c65_mgpu.log
