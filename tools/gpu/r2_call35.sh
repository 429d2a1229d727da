NADMM_DMMA_VERBOSE=1 timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c35_hv.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2c35_bench.json 2> gpurun_out/r2c35_bench.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2c35_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c35_tests.log
