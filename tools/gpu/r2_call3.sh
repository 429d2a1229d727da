timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "dense_model_ops" > gpurun_out/r2c3_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c3_tests.log
NADMM_GEMM_VERBOSE=1 timeout 600 python tools/prof/hv_configs.py 5 > gpurun_out/r2c3_hv.log 2>&1
