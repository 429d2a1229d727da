set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2c2_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2c2_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2c2_bench.json 2> gpurun_out/r2c2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2c2_ref.json 2> gpurun_out/r2c2_ref.err
