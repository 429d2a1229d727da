timeout 900 python tools/dbg/gemm_race.py > gpurun_out/r2c13_dbg.log 2>&1
timeout 900 python tools/dbg/cfg5_hv2.py 40000 125000 >> gpurun_out/r2c13_dbg.log 2>&1
