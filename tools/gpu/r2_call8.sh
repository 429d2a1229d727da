timeout 1800 python -m pytest tests/test_scale.py -x -q --durations=0 > gpurun_out/r2c8_scale.log 2>&1
echo "rc=$?" >> gpurun_out/r2c8_scale.log
timeout 300 python tools/prof/hv_configs.py 4 > gpurun_out/r2c8_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__t_bytes.sum --clock-control none -k regex:"sparse|transpose" -c 24 --csv --log-file gpurun_out/r2c8_sparse_launches.csv python tools/prof/hv_configs.py 4 > gpurun_out/r2c8_ncu.log 2>&1
