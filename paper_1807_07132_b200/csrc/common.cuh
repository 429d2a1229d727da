// Shared device/host helpers for the Newton-ADMM sm_100a library.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
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
constexpr int kCscQuad = 4;        // CSC columns of the lane-group path are padded to multiples of this
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

// Software grid barrier for kernels whose whole grid is co-resident (persistent grids launched
// cooperatively where the runtime allows it, else sized from occupancy). `ctr` is a monotonically
// increasing per-kernel counter that only launches of the same grid size touch, so it is a multiple
// of gridDim.x whenever such a launch starts; every block must reach every barrier (callers branch
// only on grid-uniform values).
//
// Watchdog (opt-out): a grid that is not fully co-resident would spin forever. After
// NADMM_BARRIER_TIMEOUT_MS of wall time (%globaltimer; default 60 s, 0 = off) the waiting block sets
// the translation unit's fault flag and every barrier of the launch falls through; the host raises
// NADMM_ECUDA at its next synchronisation (stream_sync) instead of the context dying on a trap.
struct BarrierCtl {
    unsigned long long timeout_ns;
    unsigned long long fault;
};
struct BarrierTU {
    void (*set_timeout)(unsigned long long ns);
    unsigned long long (*take_fault)();
};
void barrier_register(BarrierTU tu);  // host registry (newton.cu): one entry per translation unit

namespace {
// Without relocatable device code every translation unit owns its copy of the control block; each
// registers its accessors at static-initialisation time.
__device__ BarrierCtl g_barrier_ctl = {0ull, 0ull};

void barrier_set_timeout_tu(unsigned long long ns) {
    const BarrierCtl c{ns, 0ull};
    cudaMemcpyToSymbol(g_barrier_ctl, &c, sizeof c);
}

unsigned long long barrier_take_fault_tu() {
    BarrierCtl c{};
    if (cudaMemcpyFromSymbol(&c, g_barrier_ctl, sizeof c) != cudaSuccess) return 0;
    if (c.fault) {
        c.fault = 0;
        cudaMemcpyToSymbol(g_barrier_ctl, &c, sizeof c);
    }
    return c.fault ? 1ull : 0ull;
}

struct BarrierReg {
    BarrierReg() { barrier_register(BarrierTU{barrier_set_timeout_tu, barrier_take_fault_tu}); }
} g_barrier_reg;
}  // namespace

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Barrier over `nb` co-resident blocks that share the counter (the whole grid, or a sub-grid).
__device__ __forceinline__ void grid_barrier_n(unsigned long long* ctr, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long nb = nblocks;
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ULL);
        const unsigned long long target = (old / nb + 1) * nb;
        const unsigned long long limit = g_barrier_ctl.timeout_ns;
        const unsigned long long t0 = limit ? global_ns() : 0ull;
        unsigned long long cur;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(cur) : "l"(ctr) : "memory");
            if (cur >= target) break;
            if (limit) {
                if (*(volatile unsigned long long*)&g_barrier_ctl.fault) break;  // an earlier barrier timed out
                if (global_ns() - t0 > limit) {
                    atomicExch(&g_barrier_ctl.fault, 1ull);
                    break;
                }
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned long long* ctr) { grid_barrier_n(ctr, gridDim.x); }

// Persistent grids that synchronise through grid_barrier are launched cooperatively (the runtime
// then guarantees co-residency, or fails the launch); NADMM_COOP=0 falls back to plain launches
// (co-residency from the occupancy-sized grid, guarded by the barrier watchdog).
inline bool coop_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("NADMM_COOP");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_ex(bool coop, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (coop && coop_enabled()) ? 1 : 0;
    NADMM_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    launch_ex(false, kernel, grid, block, smem, st, args...);
}

// Grid-barrier kernels (grid_barrier inside): cooperative launch.
template <typename... KArgs, typename... Args>
void launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    launch_ex(true, kernel, grid, block, smem, st, args...);
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace nadmm
