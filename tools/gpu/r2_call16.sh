NADMM_DMMA_VERBOSE=1 timeout 600 python bench.py --no-cpu --no-ttt --steps 3 > gpurun_out/r2c16_plain.json 2> gpurun_out/r2c16_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:dmma_group -s 40 -c 1 -o gpurun_out/r2c16_group python bench.py --no-cpu --no-ttt --steps 3 > gpurun_out/r2c16_ncu.log 2>&1
