# 16-row DMMA tiles (lag 1 / 3 stages etc.) for narrow slices: cfg1 timing and parity with the variant library
export NADMM_LIB=$PWD/tools/prof/variants/libnadmm_bm16.so
NADMM_DMMA_VERBOSE=1 timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c64_hv_bm16.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense_model_ops or newton_single" > gpurun_out/r2c64_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c64_tests.log
timeout 600 python bench.py --config cfg1 --no-cpu --no-ttt > gpurun_out/r2c64_cfg1.json 2> gpurun_out/r2c64_cfg1.err
unset NADMM_LIB
timeout 600 python bench.py --config cfg1 --no-cpu --no-ttt > gpurun_out/r2c64_cfg1_base.json 2> gpurun_out/r2c64_cfg1_base.err
