timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2c7_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c7_tests.log
timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c7_bench.json 2> gpurun_out/r2c7_bench.err
