# phase B without the row mask on full tiles
timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c48_hv.txt 2>&1
timeout 300 python tools/prof/graph_timeline.py > gpurun_out/r2c48_tl.txt 2>&1
timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c48_bench.json 2> gpurun_out/r2c48_bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale.py -m gpu -q -x > gpurun_out/r2c48_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c48_tests.log
