// TMA / mbarrier / DMMA primitives shared by the tensor-map kernels (kernels_gemm.cu, kernels_sparse.cu),
// plus the host-side tensor-map encoder (cuTensorMapEncodeTiled through the runtime's driver entry
// point, so the library needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"

namespace nadmm {
namespace tma {

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}

__device__ __forceinline__ void fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}

// 2-D tiled tensor load (SASS UTMALDG) into shared memory, completing its bytes on `bar`.
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// FP64 tensor-core MMA m8n8k4 (SASS DMMA.8x8x4): c += a * b. Fragments: a = A[gq][tq] (row-major
// 8x4), b = B[tq][gq] (4x8), c = C[gq][2tq], C[gq][2tq+1], with gq = lane / 4, tq = lane % 4.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// Byte offset of element (row, col) in a [rows][16 doubles] tile written by TMA with 128-byte
// swizzle (16-byte chunk index XOR row mod 8; the tile must be 1024-byte aligned).
__host__ __device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t col) {
    return row * 128u + ((((col >> 1) ^ (row & 7u)) << 4) | ((col & 1u) << 3));
}

// Host: a 2-D FP64 tensor map over a row-major matrix (inner = contiguous extent in elements, outer
// = rows, row_bytes = leading dimension in bytes, a multiple of 16), box {box_inner, box_outer},
// 128-byte swizzle (box_inner * 8 <= 128), out-of-bounds elements read as zero.
CUtensorMap make_map_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                        uint32_t box_outer);

}  // namespace tma
}  // namespace nadmm
