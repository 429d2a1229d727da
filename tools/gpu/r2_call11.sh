timeout 900 python tools/dbg/cfg5_hv2.py > gpurun_out/r2c11_dbg.log 2>&1
NADMM_DISABLE_GEMM=1 timeout 900 python tools/dbg/cfg5_hv2.py 125000 >> gpurun_out/r2c11_dbg.log 2>&1
