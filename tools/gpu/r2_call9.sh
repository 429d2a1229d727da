NADMM_GEMM_VERBOSE=1 timeout 900 python tools/dbg/gemm_hv_sizes.py > gpurun_out/r2c9_dbg.log 2>&1
