timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c34_bench.json 2> gpurun_out/r2c34_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2c34_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c34_tests.log
