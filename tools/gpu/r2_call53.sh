timeout 1500 python -m pytest tests/test_scale.py -m gpu -q -k "workers_round or lbfgs_worker" > gpurun_out/r2c53_scale.log 2>&1; echo "rc=$?" >> gpurun_out/r2c53_scale.log
