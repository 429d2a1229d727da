# handle-lifetime tests; full GPU suite; e2e split at N=4 is a separate call
timeout 600 python -m pytest tests/test_lifetime.py -m gpu -q -x > gpurun_out/r2c38_life.log 2>&1; echo "rc=$?" >> gpurun_out/r2c38_life.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2c38_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c38_tests.log
# in-bench capture of the quarter-GPU Hv launch (cooperative attribute off: ncu cannot replay a
# cooperative launch inside a graph)
NADMM_COOP=0 CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_pass_kernel --launch-skip 300 -c 1 -o gpurun_out/r2c38_bench_dmma python bench.py --no-cpu --no-ttt --steps 2 --warmup 3 > gpurun_out/r2c38_ncu.log 2>&1
