# bench line with the theta <= 1e-3 leg (N=1, with the CPU parity leg)
timeout 1200 python bench.py > gpurun_out/r2c57_bench.json 2> gpurun_out/r2c57_bench.err
