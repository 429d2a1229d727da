timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2c14_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c14_tests.log
timeout 900 python tools/dbg/cfg5_hv2.py 40000 125000 > gpurun_out/r2c14_dbg.log 2>&1
