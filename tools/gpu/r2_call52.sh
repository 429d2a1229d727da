# remainder-class DFMAs as bursts after the DMMAs vs interleaved
for v in burst interleaved; do
  if [ $v = interleaved ]; then export NADMM_LIB=$PWD/tools/prof/variants/libnadmm_interleaved.so; else unset NADMM_LIB; fi
  timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c52_hv_$v.txt 2>&1
  timeout 300 python tools/prof/graph_timeline.py > gpurun_out/r2c52_tl_$v.txt 2>&1
  timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c52_bench_$v.json 2> gpurun_out/r2c52_bench_$v.err
done
unset NADMM_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale.py -m gpu -q -x > gpurun_out/r2c52_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c52_tests.log
