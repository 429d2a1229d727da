# cfg5 lambda sweep with the spectral penalty (8 x 500,000 x 2,048, C = 100, one B200)
timeout 1800 python tools/prof/cfg5_lambda_sweep.py 20 > gpurun_out/r2c61_cfg5_sweep.json 2> gpurun_out/r2c61_cfg5_sweep.err
