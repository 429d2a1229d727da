// Shared device/host helpers for the Newton-ADMM sm_100a library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/nadmm_cuda.h"

namespace nadmm {

// Internal error carrying an nadmm_status; converted to a return code at the C ABI.
struct Error : std::runtime_error {
    nadmm_status code;
    Error(nadmm_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(nadmm_status c, const std::string& m) { throw Error(c, m); }

#define NADMM_CUDA(call)                                                                               \
    do {                                                                                               \
        cudaError_t e__ = (call);                                                                      \
        if (e__ != cudaSuccess)                                                                        \
            ::nadmm::raise(NADMM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__) + " @" + \
                                            __FILE__ + ":" + std::to_string(__LINE__));                \
    } while (0)

#define NADMM_LAUNCH_CHECK() NADMM_CUDA(cudaGetLastError())

constexpr int kMaxClasses = 128;   // C - 1 <= kMaxClasses on the SIMT paths
constexpr int kRowPad = 32;        // extra rows allocated in row-indexed work buffers (tile over-read)
constexpr int kBlockPartials = 1024;  // max blocks writing partials in one reduction slot

// ---------------------------------------------------------------------------------------------
// Deterministic reductions. Every block writes one partial per slot; consumers reduce the partials
// with reduce_partials() executed by one full warp: lane l sums parts[l], parts[l+32], ... in
// ascending order, then a fixed xor-butterfly combines the lanes. Results are bit-identical across
// runs and across the blocks that redundantly evaluate them.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum in fixed order; result valid in thread 0. `scratch` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        r = lane < nw ? scratch[lane] : 0.0;
        r = warp_sum(r);
    }
    return r;
}

// Must be called by all 32 lanes of a warp.
__device__ __forceinline__ double reduce_partials(const double* parts, int n) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    int i = lane;
    for (; i + 96 < n; i += 128) {  // four loads in flight, additions in the same ascending order
        const double v0 = parts[i], v1 = parts[i + 32], v2 = parts[i + 64], v3 = parts[i + 96];
        s += v0;
        s += v1;
        s += v2;
        s += v3;
    }
    for (; i < n; i += 32) s += parts[i];
    return warp_sum(s);
}

// Software grid barrier for kernels whose whole grid is co-resident (small persistent grids on the
// context's stream). `ctr` is a monotonically increasing per-kernel counter that only launches of
// the same grid size touch, so it is a multiple of gridDim.x whenever such a launch starts; every
// block must reach every barrier (callers branch only on grid-uniform values).
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long nb = gridDim.x;
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ULL);
        const unsigned long long target = (old / nb + 1) * nb;
        unsigned long long cur;
        const long long t0 = clock64();
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(cur) : "l"(ctr) : "memory");
            // watchdog: a grid that is not fully co-resident would spin forever; fail the launch
            // (an error the host reports) instead of hanging the device (~4 s at 2 GHz)
            if (cur < target && clock64() - t0 > (8LL << 30)) __trap();
        } while (cur < target);
    }
    __syncthreads();
}

// Programmatic dependent launch: kernels of the Newton-iteration graph are launched with
// programmatic stream serialisation, so a kernel's launch and prologue overlap its predecessor's
// tail; every such kernel calls pdl_wait() before touching memory its predecessor writes (a no-op
// when the launch was not programmatic).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

#ifndef NADMM_PDL
#define NADMM_PDL 0  // measured: no gain on the Newton graph (kept switchable)
#endif

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = NADMM_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NADMM_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace nadmm
