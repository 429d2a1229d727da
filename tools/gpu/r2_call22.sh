timeout 300 python tools/prof/group_hv.py 1 50000 3072 > gpurun_out/r2c22.log 2>&1
timeout 300 python tools/prof/group_hv.py 8 6250 3072 >> gpurun_out/r2c22.log 2>&1
