timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_lbfgs.py tests/test_cpp_api.py -x -q > gpurun_out/r2c15_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c15_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/r2c15_bench.json 2> gpurun_out/r2c15_bench.err
NADMM_GROUP=0 timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c15_bench_nogroup.json 2> gpurun_out/r2c15_bench_nogroup.err
