// Like tma_stream.cu, but each CTA streams a column SLICE of a wide row-major matrix (the DMMA pass's
// access pattern: CTA r of a cluster-of-CS loads features [r*fs, (r+1)*fs) of every row), for grids of
// 120 (15 clusters of 8) and 148 CTAs.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t x) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(x) : "memory"); }
__device__ __forceinline__ void marr(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

__global__ void stream(const double* X, int64_t nrows, int rowd, int ld, int cs, int bm, int stages, double* out) {
  extern __shared__ __align__(128) double sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)stages * bm * rowd);
  uint64_t* empty = full + stages;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) { minit(&full[s], 1); minit(&empty[s], nw - 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  int64_t ntiles = nrows / bm;
  int cid = blockIdx.x / cs, ncl = gridDim.x / cs, crank = blockIdx.x % cs;
  int T = cid < ntiles ? (int)((ntiles - 1 - cid) / ncl + 1) : 0;
  double acc = 0;
  if (warp == nw - 1) {
    if (lane == 0) for (int i = 0; i < T; ++i) {
      int st = i % stages;
      if (i >= stages) mwait(&empty[st], ((i / stages) - 1) & 1);
      int64_t r0 = ((int64_t)cid + (int64_t)i * ncl) * bm;
      mexp(&full[st], bm * rowd * 8);
      for (int r = 0; r < bm; ++r) bulk(sm + ((size_t)st * bm + r) * rowd, X + (r0 + r) * ld + crank * rowd, rowd * 8, &full[st]);
    }
  } else {
    for (int i = 0; i < T; ++i) {
      int st = i % stages;
      mwait(&full[st], (i / stages) & 1);
      acc += sm[(size_t)st * bm * rowd + lane];
      __syncwarp();
      if (lane == 0) marr(&empty[st]);
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  size_t bytes = 2ull << 30;
  double* X; cudaMalloc(&X, bytes); cudaMemset(X, 0, bytes);
  double* out; cudaMalloc(&out, 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // {slice doubles, row stride doubles, CTAs per row group, rows per tile, stages, grid}
  int cfgs[][6] = {{384, 3072, 8, 8, 6, 120}, {384, 3072, 8, 8, 6, 148}, {384, 3072, 8, 8, 8, 120}, {384, 3072, 8, 16, 4, 120},
                   {768, 3072, 4, 8, 4, 132}, {768, 3072, 4, 8, 4, 148}, {384, 384, 1, 8, 6, 120}, {384, 384, 1, 8, 6, 148}};
  for (auto& c : cfgs) {
    int rowd = c[0], ld = c[1], cs = c[2], bm = c[3], st = c[4], grid = c[5];
    size_t smem = (size_t)st * bm * rowd * 8 + 256;
    if (smem > 220 * 1024) continue;
    int64_t nrows = bytes / 8 / ld;
    for (int w : {4, 9}) {
      stream<<<grid, 32 * w, smem>>>(X, nrows, rowd, ld, cs, bm, st, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) stream<<<grid, 32 * w, smem>>>(X, nrows, rowd, ld, cs, bm, st, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("slice %5d B of %5d B rows, cs %d, %2d rows x %d stages (%3zu KB), grid %d, %d warps: %7.1f GB/s  %s\n", rowd * 8,
             ld * 8, cs, bm, st, smem / 1024, grid, w, 5.0 * (nrows / bm) * bm * ld * 8 / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
