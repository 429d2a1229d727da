#!/usr/bin/env bash
# Builds libnadmm_cuda.so in-tree for sm_100a (B200). No GPU needed (nvcc cross-compiles).
set -euo pipefail
cd "$(dirname "$0")"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
mkdir -p build lib
FLAGS=(-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -fopenmp
       -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Xptxas -v)
SRCS=(kernels_pass kernels_vec kernels_dmma kernels_smallp kernels_gemm kernels_sparse newton lbfgs sgd capi admm data_io host_coord)
pids=()
for s in "${SRCS[@]}"; do
  "$NVCC" "${FLAGS[@]}" -c "csrc/$s.cu" -o "build/$s.o" > "build/$s.ptxas.log" 2>&1 &
  pids+=($!)
done
rc=0
for i in "${!pids[@]}"; do
  if ! wait "${pids[$i]}"; then echo "compile failed: ${SRCS[$i]}"; cat "build/${SRCS[$i]}.ptxas.log"; rc=1; fi
done
[ $rc -eq 0 ] || exit 1
"$NVCC" -shared -gencode arch=compute_100a,code=sm_100a -o lib/libnadmm_cuda.so build/*.o -lnccl -lgomp
echo "built $(pwd)/lib/libnadmm_cuda.so"
