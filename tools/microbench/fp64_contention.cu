// Latency of a dependent DADD chain / LDS+DADD chain on one warp while other warps saturate DMMA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, int iters, int dmma_warps, long long* cyc, int mode) {
  __shared__ double sm[1024];
  int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-6;
  __syncthreads();
  if (warp < dmma_warps) {
    double a = threadIdx.x * 1e-3, b = 1.0, c[4][2] = {};
    for (int it = 0; it < iters * 4; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    if (c[0][0] == 1234.0) out[0] = c[0][0];
  } else if (warp == dmma_warps) {
    double x = threadIdx.x;
    long long t0 = clock64();
    if (mode == 0) {
      for (int it = 0; it < iters; ++it) x = x + 1e-9;       // dependent DADD chain
    } else if (mode == 1) {
      for (int it = 0; it < iters; ++it) x = x * 1.0000001 + 1e-9;  // dependent DFMA chain
    } else {
      int idx = threadIdx.x & 31;
      for (int it = 0; it < iters; ++it) { x += sm[idx]; idx = (idx + (int)x) & 1023; }  // LDS + DADD chain
    }
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cyc[0] = t1 - t0;
    if (x == 1234.0) out[0] = x;
  }
}

int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  int iters = 2000;
  const char* names[] = {"DADD chain", "DFMA chain", "LDS+DADD chain"};
  for (int mode = 0; mode < 3; ++mode)
    for (int dw : {0, 2, 4, 8}) {
      k<<<1, 32 * (dw + 1)>>>(out, iters, dw, cyc, mode);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-15s with %d DMMA warps/SM: %.1f cycles per dependent op\n", names[mode], dw, (double)h / iters);
    }
  return 0;
}
