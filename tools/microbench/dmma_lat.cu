// DMMA (mma.sync m8n8k4 f64) latency / throughput vs. independent chains and warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void chains(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
void run(int warps, double* out, long long* cyc) {
  int iters = 2000;
  chains<CH><<<1, 32 * warps>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  chains<CH><<<1, 32 * warps>>>(out, iters, cyc);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (iters * CH);
  printf("warps/SM=%2d chains/warp=%d: %.2f cyc per DMMA per warp; SM rate %.2f cyc/DMMA (%.1f FMA/clk/SM)\n",
         warps, CH, per, per / warps, 256.0 * warps / per);
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 16}) { run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); }
  return 0;
}
