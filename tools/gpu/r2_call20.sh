timeout 300 python tools/prof/group_hv.py 2 25000 3072 > gpurun_out/r2c20.log 2>&1
NADMM_COOP=0 timeout 300 python tools/prof/group_hv.py 2 25000 3072 >> gpurun_out/r2c20.log 2>&1
NADMM_COOP=0 timeout 300 python tools/prof/group_hv.py 8 6250 3072 >> gpurun_out/r2c20.log 2>&1
timeout 300 python tools/prof/group_hv.py 1 50000 3072 >> gpurun_out/r2c20.log 2>&1
