# epilogue warp count: 1 / 2 (production) / 3
for v in epi1 epi3 prod; do
  if [ $v = prod ]; then unset NADMM_LIB; else export NADMM_LIB=$PWD/tools/prof/variants/libnadmm_$v.so; fi
  timeout 300 python tools/prof/hv_configs.py 1 2 > gpurun_out/r2c68_hv_$v.txt 2>&1
  timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c68_bench_$v.json 2> gpurun_out/r2c68_bench_$v.err
done
