timeout 300 python tools/prof/group_hv.py 8 6250 3072 > gpurun_out/r2c18.log 2>&1
timeout 300 python tools/prof/group_hv.py 2 25000 3072 >> gpurun_out/r2c18.log 2>&1
timeout 300 python tools/prof/group_hv.py 8 7500 784 >> gpurun_out/r2c18.log 2>&1
