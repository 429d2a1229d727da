# cost of the cooperative launch attribute on the fused passes (timeline + bench), default vs NADMM_COOP=0
for v in coop nocoop; do
  if [ $v = nocoop ]; then export NADMM_COOP=0; else unset NADMM_COOP; fi
  timeout 300 python tools/prof/graph_timeline.py > gpurun_out/r2c55_tl_$v.txt 2>&1
  timeout 600 python bench.py --no-cpu --no-ttt > gpurun_out/r2c55_bench_$v.json 2> gpurun_out/r2c55_bench_$v.err
done
