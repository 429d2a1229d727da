# per-config bench lines (BASELINE.json configs 1, 3, 4, 5) at N = 1
for c in cfg1 cfg3 cfg4; do
  timeout 1200 python bench.py --config $c > gpurun_out/r2c24_$c.json 2> gpurun_out/r2c24_$c.err
done
timeout 2400 python bench.py --config cfg5 --steps 5 > gpurun_out/r2c24_cfg5.json 2> gpurun_out/r2c24_cfg5.err
