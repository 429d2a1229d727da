timeout 300 python tools/prof/group_hv.py 8 6250 3072 > gpurun_out/r2c19.log 2>&1
timeout 300 python tools/prof/group_hv.py 2 25000 3072 >> gpurun_out/r2c19.log 2>&1
timeout 300 python tools/prof/group_hv.py 8 7500 784 >> gpurun_out/r2c19.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_lbfgs.py -x -q > gpurun_out/r2c19_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c19_tests.log
timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c19_bench.json 2> gpurun_out/r2c19_bench.err
