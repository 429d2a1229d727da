timeout 300 python tools/prof/group_hv.py 8 6250 3072 > gpurun_out/r2c33.log 2>&1
NADMM_GROUP_CONTIG=1 timeout 300 python tools/prof/group_hv.py 8 6250 3072 >> gpurun_out/r2c33.log 2>&1
NADMM_GROUP=1 NADMM_GROUP_CONTIG=1 timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c33_bench_contig.json 2> gpurun_out/r2c33_bench_contig.err
NADMM_GROUP=1 timeout 900 python bench.py --no-cpu --no-ttt > gpurun_out/r2c33_bench_strided.json 2> gpurun_out/r2c33_bench_strided.err
