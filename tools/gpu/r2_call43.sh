# CSR rows pass in Hv mode: blocks per SM 8 (production) / 16 / 32 / 64
for b in 8 16 32 64; do NADMM_SP_HV_BPS=$b timeout 300 python tools/prof/hv_configs.py 4 > gpurun_out/r2c43_bps$b.txt 2>&1; done
