NADMM_GROUP=1 timeout 900 python bench.py --no-cpu > gpurun_out/r2c29_group.json 2> gpurun_out/r2c29_group.err
timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c29_streams.json 2> gpurun_out/r2c29_streams.err
