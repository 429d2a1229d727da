# node-group kernel vs single-pass kernel on the same 50,000 x 3,072 shard (no tails): ncu --set full of one launch each
timeout 300 python tools/prof/group_hv.py 1 50000 > gpurun_out/r2c47_group_1x50000.txt 2>&1
timeout 300 python tools/prof/group_hv.py 8 6250 > gpurun_out/r2c47_group_8x6250.txt 2>&1
NADMM_COOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_group_kernel --launch-skip 2 -c 1 -o gpurun_out/r2c47_group python tools/prof/group_hv.py 1 50000 > gpurun_out/r2c47_ncu_group.log 2>&1
NADMM_COOP=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma_pass_kernel<8, 1, 1, 8, 2, 5, 1>" --launch-skip 2 -c 1 -o gpurun_out/r2c47_pass python tools/prof/group_hv.py 1 50000 > gpurun_out/r2c47_ncu_pass.log 2>&1
