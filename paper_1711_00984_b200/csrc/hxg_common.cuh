// hxg_common.cuh -- device constants and intrinsics shared by all kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "hxg_plan.h"

#ifndef HXG_DMMA_KEEP
#define HXG_DMMA_KEEP 0
#endif

namespace hxg {

constexpr int GEN_THREADS = 256;
constexpr int GEN_WARPS = GEN_THREADS / 32;

// FP64 tensor-core MMA, D(8x8) += A(8x4, row) * B(4x8, col); lowers to DMMA.8x8x4.
// Fragments: A[g][t], B[t][g], D[g][2t + {0,1}] with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// Same MMA, but the A operand stays live afterwards (an integer use folded into
// `keep`), so the register allocator cannot place the destination D on top of
// A.  ptxas for sm_100a was observed to emit DMMA with D overlapping A and the
// result was wrong (tools/dbg_v3.cu); keeping A live avoids that allocation.
__device__ __forceinline__ void dmma_8x8x4_keep(double &d0, double &d1, double a, double b, unsigned &keep)
{
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
#if HXG_DMMA_KEEP
    keep ^= (unsigned)__double2loint(a) + (unsigned)__double2loint(b);
#else
    (void)keep;
#endif
}

}  // namespace hxg
