timeout 900 python tools/prof/ttt_1e3.py > gpurun_out/r2c56_ttt.txt 2>&1
