// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput and HBM read bandwidth on B200.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(in + i); s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float ms;
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 4000;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("DFMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
    dmma_kernel<<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
  }
  size_t bytes = 4ull << 30; double2* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  for (int bpsm : {2, 4, 8}) {
    read_kernel<<<sms * bpsm, 512>>>(buf, bytes / 16, out); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); read_kernel<<<sms * bpsm, 512>>>(buf, bytes / 16, out); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("HBM read blocks/SM=%d: %.1f GB/s\n", bpsm, bytes / best / 1e6);
  }
  return 0;
}
