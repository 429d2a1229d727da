timeout 1500 python tools/dbg/cfg5_hv.py > gpurun_out/r2c10_dbg.log 2>&1
/tmp/l2_bw > /dev/null 2>&1; nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench/l2_bw tools/microbench/l2_bw.cu && tools/microbench/l2_bw > gpurun_out/r2c10_l2bw.log 2>&1
