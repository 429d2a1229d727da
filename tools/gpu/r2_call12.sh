timeout 900 python tools/dbg/gemm_race.py > gpurun_out/r2c12_dbg.log 2>&1
NADMM_GEMM_POISON_U=1 timeout 900 python tools/dbg/gemm_race.py >> gpurun_out/r2c12_dbg.log 2>&1
