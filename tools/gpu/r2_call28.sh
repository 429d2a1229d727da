NADMM_DMMA_AUTOTUNE=0 timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/dbg/sanitize_dmma.py > gpurun_out/r2c28_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/r2c28_racecheck.log
