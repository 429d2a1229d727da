timeout 300 python tools/prof/group_hv.py 8 6250 3072 > gpurun_out/r2c27.log 2>&1
timeout 300 python tools/prof/group_hv.py 1 50000 3072 >> gpurun_out/r2c27.log 2>&1
timeout 900 python bench.py --config cfg1 > gpurun_out/r2c27_cfg1.json 2> gpurun_out/r2c27_cfg1.err
