timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "repeatable or dense_model_ops or admm" > gpurun_out/r2c30_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c30_tests.log
NADMM_DMMA_VERBOSE=1 timeout 600 python tools/prof/hv_configs.py 1 2 3 4 5 > gpurun_out/r2c30_hv.log 2>&1
