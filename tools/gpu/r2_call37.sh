# alternating-direction DMMA passes (L2 reuse between consecutive passes) vs forward-only
for m in fwd snake; do
  if [ $m = fwd ]; then export NADMM_DMMA_FORWARD=1; else unset NADMM_DMMA_FORWARD; fi
  timeout 300 python tools/prof/graph_timeline.py > gpurun_out/r2c37_tl_$m.txt 2>&1
  timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c37_bench_$m.json 2> gpurun_out/r2c37_bench_$m.err
done
unset NADMM_DMMA_FORWARD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale.py -m gpu -q -x > gpurun_out/r2c37_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c37_tests.log
