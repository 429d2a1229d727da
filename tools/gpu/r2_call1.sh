nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2c1_smi.txt
lscpu > gpurun_out/r2c1_lscpu.txt; nproc > gpurun_out/r2c1_nproc.txt
timeout 300 python tools/prof/fp64_peak.py gpurun_out/r2_fp64_peak.json > gpurun_out/r2c1_fp64.log 2>&1
timeout 600 python tools/prof/hv_configs.py 1 2 3 4 5 > gpurun_out/r2c1_hv.log 2>&1
