# reference arm with both time-to-target thresholds on the GPU box's host cores
timeout 1200 python bench.py --impl reference > gpurun_out/r2c58_ref.json 2> gpurun_out/r2c58_ref.err
nproc > gpurun_out/r2c58_nproc.txt
