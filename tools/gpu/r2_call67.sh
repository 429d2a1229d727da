# final full GPU suite on 2 GPUs + smoke
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2c67_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c67_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2c67_smoke.log 2>&1
