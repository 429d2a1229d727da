# launch list of the bench command (per-launch device time + DRAM bytes; serialised by ncu)
NADMM_COOP=0 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2c62_launches.csv python bench.py --no-cpu --no-ttt --steps 2 --warmup 3 > gpurun_out/r2c62_ncu.log 2>&1
gzip -kf gpurun_out/r2c62_launches.csv
