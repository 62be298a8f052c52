// hxg_device.h -- host-side device queries shared by every launcher.
//
// Grid heuristics size persistent grids as a multiple of the SM count of the
// CURRENT device (148 on B200) instead of a hard-coded constant.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

namespace hxg {

// Number of SMs of the current device (cached per device ordinal; thread-safe).
inline int sm_count()
{
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    int v = cache[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

// Highest isotropic order served by a kernel that evaluates the element geometry itself
// (no metric pass / workspace): the low-order slab kernel general_lo_kernel covers
// p <= 4; HXG_LO=0 falls back to the fused warp-unit kernel (p <= 3).
inline int fused_order_max()
{
    const char *v = getenv("HXG_LO");
    return (v && v[0] == '0') ? 3 : 4;
}

}  // namespace hxg
