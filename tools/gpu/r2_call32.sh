timeout 1200 python -m pytest tests/test_group.py -x -q > gpurun_out/r2c32_group.log 2>&1
echo "rc=$?" >> gpurun_out/r2c32_group.log
timeout 900 python bench.py > gpurun_out/r2c32_bench.json 2> gpurun_out/r2c32_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2c32_ref.json 2> gpurun_out/r2c32_ref.err
