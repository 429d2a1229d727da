# per-config lines after the last bench edits (cfg1 with ttt, cfg3), smoke
timeout 900 python bench.py --config cfg1 > gpurun_out/r2c63_cfg1.json 2> gpurun_out/r2c63_cfg1.err
timeout 900 python bench.py --config cfg3 > gpurun_out/r2c63_cfg3.json 2> gpurun_out/r2c63_cfg3.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2c63_smoke.log 2>&1
