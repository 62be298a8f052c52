// hxg_common.cuh -- device constants and intrinsics shared by all kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "hxg_plan.h"

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

}  // namespace hxg
