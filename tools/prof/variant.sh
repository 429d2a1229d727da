#!/bin/bash
# Build a variant of libnadmm_cuda.so with extra nvcc defines for the DMMA pass only:
#   tools/prof/variant.sh NAME -DFOO=1 ...   ->  tools/prof/var_NAME.so  (run with NADMM_LIB=...)
# Needs a prior paper_1807_07132_b200/build.sh (reuses its other objects).
set -e
cd "$(dirname "$0")/../../paper_1807_07132_b200"
name=$1; shift
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
mkdir -p /tmp/var_$name
"$NVCC" -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Xptxas -v "$@" -c csrc/kernels_dmma.cu -o /tmp/var_$name/kernels_dmma.o > /tmp/var_$name/ptxas.log 2>&1 || { tail -20 /tmp/var_$name/ptxas.log; exit 1; }
for o in build/*.o; do [ "$(basename $o)" = kernels_dmma.o ] || cp $o /tmp/var_$name/; done
"$NVCC" -shared -gencode arch=compute_100a,code=sm_100a -o ../tools/prof/var_$name.so /tmp/var_$name/*.o -lnccl
echo "built tools/prof/var_$name.so"
