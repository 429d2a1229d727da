timeout 2400 python -m pytest tests/test_scale.py -x -q --durations=0 > gpurun_out/r2c4_scale.log 2>&1
echo "rc=$?" >> gpurun_out/r2c4_scale.log
