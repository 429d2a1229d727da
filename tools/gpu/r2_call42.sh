# CSR Hv: one resident wave (occupancy-sized grid) at 64 regs vs 40 regs (6 blocks/SM)
timeout 300 python tools/prof/hv_configs.py 4 > gpurun_out/r2c42_sp_default.txt 2>&1
NADMM_LIB=$PWD/tools/prof/variants/libnadmm_sp6.so timeout 300 python tools/prof/hv_configs.py 4 > gpurun_out/r2c42_sp6.txt 2>&1
