# full verification: edge tests, whole GPU suite, smoke, N=1 bench (parity + CPU baseline + ttt), reference arm
timeout 600 python -m pytest tests/test_edges.py -m gpu -q > gpurun_out/r2c49_edges.log 2>&1; echo "rc=$?" >> gpurun_out/r2c49_edges.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2c49_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c49_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2c49_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2c49_bench.json 2> gpurun_out/r2c49_bench.err
timeout 1200 python bench.py --impl reference > gpurun_out/r2c49_ref.json 2> gpurun_out/r2c49_ref.err
