# split-role DMMA pass (phase-A and phase-B warps): timings, bench, parity
NADMM_DMMA_VERBOSE=1 timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c40_hv.txt 2>&1
timeout 300 python tools/prof/graph_timeline.py > gpurun_out/r2c40_tl.txt 2>&1
timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c40_bench.json 2> gpurun_out/r2c40_bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale.py -m gpu -q -x > gpurun_out/r2c40_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c40_tests.log
