# ncu --set full of the top kernels (one launch each): two-GEMM path (cfg5 quarter shard), dense DMMA pass (cfg2 shard)
python tools/prof/hv_configs.py 5 > gpurun_out/r2c25_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_rows -s 2 -c 1 -o gpurun_out/r2c25_gemm_rows python tools/prof/hv_configs.py 5 > gpurun_out/r2c25_ncu_rows.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_xtu -s 2 -c 1 -o gpurun_out/r2c25_gemm_xtu python tools/prof/hv_configs.py 5 > gpurun_out/r2c25_ncu_xtu.log 2>&1
python tools/prof/hv_configs.py 2 > gpurun_out/r2c25_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dmma_pass -s 5 -c 1 -o gpurun_out/r2c25_dmma python tools/prof/hv_configs.py 2 > gpurun_out/r2c25_ncu_dmma.log 2>&1
