timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2c6_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c6_tests.log
timeout 600 python tools/prof/hv_configs.py 4 5 > gpurun_out/r2c6_hv.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/r2c6_bench.json 2> gpurun_out/r2c6_bench.err
