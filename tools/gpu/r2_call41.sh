# full ncu capture of the two CSR Hv kernels at the cfg4 shard (one launch each)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sparse_rows_kernel|sparse_cols_kernel" --launch-skip 2 -c 2 -o gpurun_out/r2c41_sparse python tools/prof/hv_configs.py 4 > gpurun_out/r2c41_ncu.log 2>&1
