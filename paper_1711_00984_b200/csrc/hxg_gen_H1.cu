#include <algorithm>
#include <cstdlib>
// Specialized general-map kernels for space H1, isotropic orders p = 1..10, L = p + 1.
#include "hxg_general_v2.cuh"
#include "hxg_general_v3.cuh"
#include "hxg_general_v4.cuh"
#include "hxg_affine_v2.cuh"
#include "hxg_extrusion.cuh"
#include "hxg_v2_launch.h"

namespace hxg {

template <int P>
static int launch_one(const V2Args &a, int grid, cudaStream_t st)
{
    using C4 = V4Cfg<H1, P, P + 1>;
    if constexpr (C4::OK && P >= 5) {
        const char *v4env = getenv("HXG_USE_V4");
        const bool use_v4 = v4env && v4env[0] == '1';  // opt-in: v2 measures faster at p >= 8
        if (use_v4 && !(getenv("HXG_FORCE_V2") && getenv("HXG_FORCE_V2")[0] == '1')) {
            auto k4 = general_v4_kernel<H1, P, P + 1>;
            if (cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, C4::SMEM_BYTES) != cudaSuccess)
                return -5;
            V3Args b;
            b.tables = a.tables;
            b.metric = a.metric;
            b.out = a.out;
            b.P = a.P;
            b.E = a.E;
            b.kind = nullptr;
            b.params = b.coef = b.wgrid = nullptr;
            b.status = nullptr;
            const int want = 148 * C4::MINB * 4;
            b.split = a.E >= want ? 1 : (want + a.E - 1) / a.E;
            if (b.split > 32) b.split = 32;
            k4<<<a.E * b.split, C4::THREADS, C4::SMEM_BYTES, st>>>(b);
            return cudaGetLastError() == cudaSuccess ? 0 : -5;
        }
    }
    using C3 = V3Cfg<H1, P, P + 1>;
    // general_v3_kernel<H1, 7, 8> is miscompiled by ptxas -O3 (CUDA 12.9; wrong
    // results that change with unrelated dead code, correct at -Xptxas -O0;
    // repro: tools/dbg_v3.cu) -- p = 7 runs the CTA-chunked v2 kernel instead.
    if constexpr (C3::OK && P != 7) {
        // fused kernels (p <= 3) evaluate the geometry themselves: they take the
        // fused call (metric == NULL); a call with a metric array runs v2
        if (!(getenv("HXG_FORCE_V2") && getenv("HXG_FORCE_V2")[0] == '1') &&
            (C3::FUSED == (a.metric == nullptr))) {
            auto k3 = general_v3_kernel<H1, P, P + 1>;
            if (cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, C3::SMEM_BYTES) != cudaSuccess)
                return -5;
            V3Args b;
            b.tables = a.tables;
            b.metric = a.metric;
            b.out = a.out;
            b.P = a.P;
            b.E = a.E;
            b.kind = a.kind;
            b.params = a.params;
            b.coef = a.coef;
            b.wgrid = a.wgrid;
            b.status = a.status;
            // one element per item once the batch fills a wave of CTAs: the warps then
            // flow from element to element (general_v3_kernel, HXG_V3_FLOW)
            const int want = 148 * C3::MINB * 2;
            b.split = a.E >= 148 * C3::MINB ? 1 : (want + a.E - 1) / a.E;
            if (b.split > 16) b.split = 16;
            if (getenv("HXG_V3_SPLIT")) b.split = atoi(getenv("HXG_V3_SPLIT"));
            // persistent CTAs (grid-stride over (element, part) items)
            const long long items = (long long)a.E * b.split;
            const int grid = (int)std::min<long long>(items, 148LL * C3::MINB * 2);
            k3<<<grid, V3_THREADS, C3::SMEM_BYTES, st>>>(b);
            return cudaGetLastError() == cudaSuccess ? 0 : -5;
        }
    }
    using C = V2Cfg<H1, P, P + 1>;
    auto k = general_v2_kernel<H1, P, P + 1>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
        return -5;
    k<<<grid, V2_THREADS, C::SMEM_BYTES, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

template <int P>
static int units_one() { return V2Cfg<H1, P, P + 1>::NU; }

// returns 1 if no specialization exists for p, else 0 / negative error
int launch_v2_H1(int p, const V2Args &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return launch_one<PP>(a, a.E * units_one<PP>(), st);
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#undef HXG_CASE
    }
    return 1;
}

template <int P>
static int launch_aff_one(const AffV2Args &a, cudaStream_t st)
{
    using C = AffCfg<H1, P>;
    if constexpr (C::SMEM_BYTES > 200 * 1024) {
        return 1;  // row images do not fit: runtime-generic affine kernel
    }
    auto k = affine_v2_kernel<H1, P>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
        return -5;
    // low orders with many elements: one CTA per element (row groups are tiny);
    // otherwise one CTA per packed row group
    AffV2Args b = a;
    b.rg = aff_row_groups(C::NU, a.P, a.E);
    const long long grid = (long long)a.E * ((C::NU + b.rg - 1) / b.rg);
    if (grid >= (1ll << 31)) return -6;
    k<<<(int)grid, AFF2_THREADS, C::SMEM_BYTES, st>>>(b);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// specialized constant-Jacobian kernel; returns 1 if none exists for p
int launch_aff_H1(int p, const AffV2Args &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return launch_aff_one<PP>(a, st);
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#undef HXG_CASE
    }
    return 1;
}

// specialized extrusion-map kernel (simp_*_ext); returns 1 if none exists for p
int launch_ext_H1(int p, const ExtArgs &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return launch_ext_t<H1, PP>(a, st);
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#undef HXG_CASE
    }
    return 1;
}

}  // namespace hxg
