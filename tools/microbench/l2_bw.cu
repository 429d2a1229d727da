// L2 throughput on B200: every SM repeatedly reads an L2-resident buffer (sizes below the 126 MB L2)
// with 16-byte loads, plus a gather variant (random 160-byte rows of a 40 MB table, the sparse Hv's
// access pattern). The denominator of the sparse passes' L2 roofline (they are L2 -> SM bound).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stream_read(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 1234.5) out[0] = s;
}

// 10 lanes x 16 B = one 160-byte row per group of 10 lanes, 3 groups per warp, random rows
__global__ void gather_rows(const double2* __restrict__ tab, int rows, long long items, double* out) {
  const int lane = threadIdx.x & 31, grp = lane / 10, sub = lane % 10;
  unsigned long long x = 88172645463325252ull ^ (blockIdx.x * 1315423911ull + threadIdx.x / 32);
  double s = 0;
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long it = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; it < items; it += warps) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const int r = (int)((x >> 20) % (unsigned long long)rows);
    const int rr = __shfl_sync(0xffffffffu, r + grp * 7919, 0) % rows;
    if (grp < 3) {
      double2 v = __ldg(tab + (size_t)rr * 10 + sub);
      s += v.x + v.y;
    }
  }
  if (s == 1234.5) out[0] = s;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t mb : {16, 32, 64}) {
    size_t n = (mb << 20) / 16;
    double2* a; cudaMalloc(&a, n * 16); cudaMemset(a, 0, n * 16);
    for (int bpsm : {4, 8}) {
      stream_read<<<sms * bpsm, 512>>>(a, n, 2, out);
      cudaEventRecord(e0);
      stream_read<<<sms * bpsm, 512>>>(a, n, 20, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("L2 stream read %3zu MB, %d blocks/SM: %.0f GB/s\n", mb, bpsm, 20.0 * n * 16 / (ms * 1e-3) / 1e9);
    }
    cudaFree(a);
  }
  int rows = 250000;  // 40 MB table of 160-byte rows
  double2* tab; cudaMalloc(&tab, (size_t)rows * 160); cudaMemset(tab, 0, (size_t)rows * 160);
  long long items = 20000000;
  for (int bpsm : {4, 8}) {
    gather_rows<<<sms * bpsm, 256>>>(tab, rows, items / 10, out);
    cudaEventRecord(e0);
    gather_rows<<<sms * bpsm, 256>>>(tab, rows, items, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("L2 gather 160-B rows (3 per warp step), %d blocks/SM: %.0f GB/s of rows\n", bpsm,
           items * 3.0 * 160 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
