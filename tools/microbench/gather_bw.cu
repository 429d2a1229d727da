// Random-row gather throughput from an L2-resident table on B200: the access pattern of the sparse Hv
// passes (one 160-byte K = 19 row per nonzero, rows chosen by a precomputed random index stream, as in
// a CSR/CSC index array). Many independent gathers in flight per lane (UNR), 16-byte (VW = 2) or
// 32-byte (VW = 4, sm_100 256-bit) words, tables of 20 MB (the U table of a cfg4 shard) and 42 MB (one
// column block of transposed weights). The denominator of the sparse passes' roofline.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int VW>
__device__ __forceinline__ void ldw(const double* p, double (&o)[VW]) {
  if constexpr (VW == 4) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  } else {
    double2 t = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = t.x; o[1] = t.y;
  }
}

// Each warp walks a contiguous segment of the index stream (like a CSR row), 32 indices per chunk,
// G = 32 / L groups of L = 20 / VW lanes per row.
template <int VW, int UNR, bool VALS>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ tab, const int32_t* __restrict__ idx,
                                              const double* __restrict__ val, long long nidx, int seg, double* out) {
  constexpr int L = 20 / VW, G = 32 / L;
  const int lane = threadIdx.x & 31, grp = lane / L, sub = lane - grp * L;
  const long long warps = (long long)gridDim.x * 8;
  double acc[VW] = {};
  for (long long w = blockIdx.x * 8ll + threadIdx.x / 32; w * seg < nidx; w += warps) {
    const long long q0 = w * seg, q1 = min(nidx, q0 + seg);
    for (long long qb = q0; qb < q1; qb += 32) {
      const int cnt = (int)min(32ll, q1 - qb);
      const int jl = lane < cnt ? __ldg(idx + qb + lane) : 0;
      const double vl = (VALS && lane < cnt) ? __ldg(val + qb + lane) : 1.0;
      for (int t = 0; t < cnt; t += G * UNR) {
        double v[UNR][VW], vv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int k = t + u * G + grp;
          const int jj = __shfl_sync(0xffffffffu, jl, k & 31);
          vv[u] = VALS ? __shfl_sync(0xffffffffu, vl, k & 31) : 1.0;
          if (grp < G && k < cnt) ldw<VW>(tab + (int64_t)jj * 20 + sub * VW, v[u]);
          else for (int e = 0; e < VW; ++e) v[u][e] = 0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          for (int e = 0; e < VW; ++e) acc[e] += vv[u] * v[u][e];
      }
    }
  }
  double s = 0;
  for (int e = 0; e < VW; ++e) s += acc[e];
  if (s == 1234.5) out[0] = s;
}

template <int VW, int UNR, bool VALS>
void run(const double* tab, const int32_t* idx, const double* val, long long nidx, long long total, int seg, int sms,
         double* out, const char* tag) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nwin = (int)(total / nidx);
  for (int bpsm : {4}) {
    gather<VW, UNR, VALS><<<sms * bpsm, 256>>>(tab, idx, val, nidx, seg, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) {
      const long long off = (long long)(r % nwin) * nidx;
      gather<VW, UNR, VALS><<<sms * bpsm, 256>>>(tab, idx + off, VALS ? val + off : nullptr, nidx, seg, out);
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%s VW=%d UNR=%d vals=%d windows=%d seg=%d %d blocks/SM: %.3f ms  %6.0f GB/s of rows (160 B)\n", tag, VW,
           UNR, (int)VALS, nwin, seg, bpsm, ms, nidx * 160.0 / (ms * 1e-3) / 1e9);
  }
}

// Variant without shuffles: each lane loads its nonzero's index and value itself (the group's lanes
// read the same address: one broadcast request), same interleaved nonzero-to-group assignment.
template <int VW, int UNR>
__global__ void __launch_bounds__(256, 4) gather_direct(const double* __restrict__ tab, const int32_t* __restrict__ idx,
                                                     const double* __restrict__ val, long long nidx, int seg, double* out) {
  constexpr int L = 20 / VW, G = 32 / L;
  const int lane = threadIdx.x & 31, grp = lane / L, sub = lane - grp * L;
  const bool act = grp < G;
  const long long warps = (long long)gridDim.x * 8;
  double acc[VW] = {};
  for (long long w = blockIdx.x * 8ll + threadIdx.x / 32; w * seg < nidx; w += warps) {
    const long long q0 = w * seg, q1 = min(nidx, q0 + seg);
    for (long long t = q0 + grp; t < q1; t += G * UNR) {
      int jj[UNR];
      double vv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const long long k = t + u * G;
        const bool ok = act && k < q1;
        jj[u] = ok ? __ldg(idx + k) : -1;
        vv[u] = ok ? __ldg(val + k) : 0.0;
      }
      double v[UNR][VW];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (jj[u] >= 0) ldw<VW>(tab + (int64_t)jj[u] * 20 + sub * VW, v[u]);
        else for (int e = 0; e < VW; ++e) v[u][e] = 0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        for (int e = 0; e < VW; ++e) acc[e] += vv[u] * v[u][e];
    }
  }
  double s = 0;
  for (int e = 0; e < VW; ++e) s += acc[e];
  if (s == 1234.5) out[0] = s;
}

template <int VW, int UNR>
void run_direct(const double* tab, const int32_t* idx, const double* val, long long nidx, long long total, int seg,
                int sms, double* out, const char* tag) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nwin = (int)(total / nidx);
  gather_direct<VW, UNR><<<sms * 4, 256>>>(tab, idx, val, nidx, seg, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) {
    const long long off = (long long)(r % nwin) * nidx;
    gather_direct<VW, UNR><<<sms * 4, 256>>>(tab, idx + off, val + off, nidx, seg, out);
  }
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("%s DIRECT VW=%d UNR=%d windows=%d seg=%d: %.3f ms  %6.0f GB/s of rows (160 B)\n", tag, VW, UNR, nwin, seg, ms,
         nidx * 160.0 / (ms * 1e-3) / 1e9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8);
  const long long nidx = 81250000 / 5;  // one cfg4 column block's nonzeros (~16M)
  const long long total = 81250000;     // all five blocks: a fresh (DRAM) index / value window per launch
  for (long long rows : {125000ll, 260000ll}) {  // 20 MB (U), 42 MB (a column block of weights)
    double* tab; cudaMalloc(&tab, rows * 160); cudaMemset(tab, 0, rows * 160);
    std::vector<int32_t> h(total);
    std::mt19937_64 g(1);
    for (auto& x : h) x = (int32_t)(g() % rows);
    int32_t* idx; cudaMalloc(&idx, total * 4); cudaMemcpy(idx, h.data(), total * 4, cudaMemcpyHostToDevice);
    double* val; cudaMalloc(&val, total * 8); cudaMemset(val, 0, total * 8);
    char tag[64]; snprintf(tag, sizeof tag, "table %3lld MB", rows * 160 >> 20);
    run<4, 3, false>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run_direct<4, 2>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run_direct<4, 3>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run_direct<4, 4>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run_direct<2, 4>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run_direct<4, 3>(tab, idx, val, nidx, total, 62, sms, out, tag);
    run<4, 3, true>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run<2, 4, true>(tab, idx, val, nidx, total, 130, sms, out, tag);
    run<4, 3, true>(tab, idx, val, nidx, total, 62, sms, out, tag);
    run<2, 4, true>(tab, idx, val, nidx, total, 62, sms, out, tag);
    cudaFree(tab); cudaFree(idx); cudaFree(val);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
