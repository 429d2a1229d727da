timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sparse" > gpurun_out/r2c5_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c5_tests.log
timeout 600 python tools/prof/hv_configs.py 4 > gpurun_out/r2c5_hv.log 2>&1
timeout 2400 python -m pytest tests/test_scale.py -x -q --durations=0 > gpurun_out/r2c5_scale.log 2>&1
echo "rc=$?" >> gpurun_out/r2c5_scale.log
