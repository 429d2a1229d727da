timeout 300 python tools/prof/group_hv.py 1 50000 3072 > gpurun_out/r2c21.log 2>&1
NADMM_LIB=tools/prof/var_static.so timeout 300 python tools/prof/group_hv.py 1 50000 3072 >> gpurun_out/r2c21.log 2>&1
