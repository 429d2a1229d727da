// DMMA issue microbenchmark for the fused K = 9 pass's instruction mix: how much of the FP64 tensor
// pipe can W warps per SM reach (W = 4, 8, 12, 16 -> 1..4 warps per SM sub-partition) with
//   (a) C independent m8n8k4 accumulator chains per warp (C = 1, 2, 4, 8), DMMA only;
//   (b) the same plus one DFMA per DMMA (the remainder class) and / or one LDS.64 per DMMA (the X
//       fragment from shared memory), as in phase A / phase B.
// One CTA per SM (148 CTAs), register-resident operands; prints TFLOP/s of the DMMA flops.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__device__ __forceinline__ double dfma_v(double a, double b, double c) {  // pinned in program order
  double d;
  asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}

// MIX bit 0: + LDS.64 operand, bit 1: + DFMA interleaved, bit 2: DFMAs as one burst after the DMMAs
template <int C, int MIX>
__global__ void kern(double* out, int iters) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double b = 1.0 + threadIdx.x * 1e-4, vr = 0.5 + lane * 1e-3;
  double c[C][2], r[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  const double* base = sm + (threadIdx.x >> 5) * 64 + lane;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      double a = (MIX & 1) ? base[(s * 8 + it) & 255] : (threadIdx.x * 1e-3 + s);
      dmma(c[s % C], a, b);
      if (MIX & 2) r[s & 3] = fma(a, vr, r[s & 3]);
    }
    if (MIX & 4) {
#pragma unroll
      for (int s = 0; s < 16; ++s) r[s & 3] = dfma_v(b + s, vr, r[s & 3]);
    }
  }
  double t = r[0] + r[1] + r[2] + r[3];
#pragma unroll
  for (int i = 0; i < C; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.0) out[0] = t;
}

template <int C, int MIX>
void run(int warps, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  kern<C, MIX><<<sms, 32 * warps>>>(out, 100);
  cudaEventRecord(e0);
  kern<C, MIX><<<sms, 32 * warps>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * 16 * iters * warps * (double)sms;
  printf("warps/SM %2d chains %d %-16s %6.2f TFLOP/s (DMMA flops)\n", warps, C, MIX == 3 ? "+DFMA +LDS" : MIX == 2 ? "+DFMA" : MIX == 1 ? "+LDS" : MIX == 4 ? "+DFMA burst" : MIX == 5 ? "+DFMA burst +LDS" : "DMMA only",
         flops / (ms * 1e-3) / 1e12);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w : {4, 8, 12, 16}) {
    run<2, 0>(w, out, e0, e1);
    run<4, 1>(w, out, e0, e1);
    run<4, 2>(w, out, e0, e1);
    run<4, 3>(w, out, e0, e1);
    run<4, 4>(w, out, e0, e1);
    run<4, 5>(w, out, e0, e1);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
