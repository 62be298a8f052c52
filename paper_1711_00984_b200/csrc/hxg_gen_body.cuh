// hxg_gen_body.cuh -- launchers of the compile-time specialized kernels of one
// space S (isotropic orders p = 1..10, general path with L = p + 1, the
// constant-Jacobian path and the extrusion path).  Each hxg_gen_<space>.cu
// instantiates this body for its space so the four spaces compile in parallel.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "hxg_affine_v2.cuh"
#include "hxg_device.h"
#include "hxg_extrusion.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_general_v3.cuh"
#include "hxg_general_pw.cuh"
#include "hxg_general_lo.cuh"
#include "hxg_metric.cuh"
#include "hxg_v2_launch.h"

namespace hxg {

static inline bool env_on(const char *name)
{
    const char *v = getenv(name);
    return v && v[0] == '1';
}

// general_v3_kernel<H1, 7, 8> was routed to v2 in round 1 after wrong results under
// ptxas -O3; the cause was a missing warp reconvergence before mma.sync (DESIGN.md
// "Warp reconvergence before mma.sync"), and the kernel runs by default (1.65x over v2,
// profiles/v3p7_r02.txt).  HXG_V3_P7=0 restores the v2 route.
template <int S, int P>
bool v3_enabled()
{
    if constexpr (S == H1 && P == 7) {
        const char *v = getenv("HXG_V3_P7");
        return !(v && v[0] == '0');
    }
    return true;
}

// warp-owned P-form kernel (hxg_general_pw.cuh): default for p >= 8 (digit extents
// 9-11, where the v3 8x8 tiles do not fit and v2's CTA-chunked stages stall at
// barriers) in H1, H(curl) and H(div) (profiles/sweep_r02.json); L2 keeps v2.
// HXG_PW=1 selects it for every order it supports, HXG_PW=0 never.
template <int S, int P>
bool pw_enabled()
{
    const char *v = getenv("HXG_PW");
    if (v && v[0] == '0') return false;
    if (v && v[0] == '1') return true;
    return P >= 8 && S != L2;
}

template <int S, int P>
int gen_launch_one(const V2Args &a, cudaStream_t st)
{
    using CP = PWCfg<S, P, P + 1>;
    if constexpr (CP::OK && P >= 4) {
        if (a.metric != nullptr && pw_enabled<S, P>() && !env_on("HXG_FORCE_V2")) {
            auto kp = general_pw_kernel<S, P, P + 1>;
            if (cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, CP::SMEM_BYTES) != cudaSuccess)
                return -5;
            PWArgs b;
            b.tables = a.tables;
            b.metric = a.metric;
            b.out = a.out;
            b.P = a.P;
            b.E = a.E;
            // CTA c takes the item range [c T / G, (c + 1) T / G) of the T = E * NU (element,
            // unit) items; G = one wave (measured best: H1 p8 73 % vs 60-69 % with 1-8 CTAs
            // per element left to the block scheduler), or HXG_PW_DIV CTAs per element
            const long long items = (long long)a.E * CP::NU;
            const char *dv = getenv("HXG_PW_DIV");
            const int div = dv ? atoi(dv) : 0;
            const long long wave = (long long)sm_count() * CP::MINB;
            const long long g = div > 0 ? std::max<long long>(wave, (long long)a.E * div) : wave;
            const int grid = (int)std::min<long long>(items, std::min<long long>(g, 1ll << 30));
            kp<<<grid, CP::THREADS, CP::SMEM_BYTES, st>>>(b);
            return cudaGetLastError() == cudaSuccess ? 0 : -5;
        }
    }
    // low orders, fused call (metric == NULL): the slab kernel (hxg_general_lo.cuh)
    if constexpr (P <= 4) {
        using CL = LoCfg<S, P>;
        if constexpr (CL::OK) {
            if (a.metric == nullptr && fused_order_max() >= 4) {
                auto kl = general_lo_kernel<S, P>;
                if (cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, CL::SMEM_BYTES) != cudaSuccess)
                    return -5;
                LoArgs b;
                b.tables = a.tables;
                b.out = a.out;
                b.P = a.P;
                b.E = a.E;
                b.kind = a.kind;
                b.params = a.params;
                b.coef = a.coef;
                b.wgrid = a.wgrid;
                b.status = a.status;
                const long long passes = ((long long)a.E + CL::EB - 1) / CL::EB;
                const int grid = (int)std::min<long long>(passes, (long long)sm_count() * CL::MINB * 4);
                kl<<<grid, LO_THREADS, CL::SMEM_BYTES, st>>>(b);
                return cudaGetLastError() == cudaSuccess ? 0 : -5;
            }
        }
    }
    using C3 = V3Cfg<S, P, P + 1>;
    if constexpr (C3::OK) {
        // fused kernels (p <= 3) evaluate the geometry themselves: they take the
        // fused call (metric == NULL); a call with a metric array runs v2
        const bool want_v3 = v3_enabled<S, P>();
        if (want_v3 && !env_on("HXG_FORCE_V2") && (C3::FUSED == (a.metric == nullptr))) {
            auto k3 = general_v3_kernel<S, P, P + 1>;
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
            const int sms = sm_count();
            const int want = sms * C3::MINB * 2;
            b.split = a.E >= sms * C3::MINB ? 1 : (want + a.E - 1) / a.E;
            if (b.split > 16) b.split = 16;
            if (getenv("HXG_V3_SPLIT")) b.split = atoi(getenv("HXG_V3_SPLIT"));
            // persistent CTAs (grid-stride over (element, part) items), or one wave of
            // CTAs with equal item ranges (HXG_V3_RANGE=1)
            const char *rg = getenv("HXG_V3_RANGE");
            b.range = (!C3::FUSED && b.split == 1 && rg && rg[0] == '1') ? 1 : 0;  // measured: no gain (H(curl) p6 -10 %)
            const long long items = b.range ? (long long)a.E * C3::NU : (long long)a.E * b.split;
            const int grid = (int)std::min<long long>(items, (long long)sms * C3::MINB * (b.range ? 1 : 2));
            k3<<<grid, V3_THREADS, C3::SMEM_BYTES, st>>>(b);
            return cudaGetLastError() == cudaSuccess ? 0 : -5;
        }
    }
    using C = V2Cfg<S, P, P + 1>;
    auto k = general_v2_kernel<S, P, P + 1>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES) != cudaSuccess)
        return -5;
    const long long grid = (long long)a.E * C::NU;
    if (grid >= (1ll << 31)) return -6;
    k<<<(int)grid, V2_THREADS, C::SMEM_BYTES, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

// returns 1 if no specialization exists for p, else 0 / negative error
template <int S>
int gen_launch(int p, const V2Args &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return gen_launch_one<S, PP>(a, st);
#ifdef HXG_QUICK_PS  // experiment builds (tools/variant_tu.sh): only these orders
        HXG_QUICK_PS
#else
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#endif
#undef HXG_CASE
    }
    return 1;
}

template <int S, int P>
int aff_launch_one(const AffV2Args &a, cudaStream_t st)
{
    using C = AffCfg<S, P>;
    if constexpr (C::SMEM_BYTES > 200 * 1024) {
        return 1;  // row images do not fit: runtime-generic affine kernel
    } else {
        auto k = affine_v2_kernel<S, P>;
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
}

// specialized constant-Jacobian kernel; returns 1 if none exists for p
template <int S>
int aff_launch(int p, const AffV2Args &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return aff_launch_one<S, PP>(a, st);
#ifndef HXG_QUICK_PS
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#endif
#undef HXG_CASE
    }
    return 1;
}

template <int S>
int met_launch(int L, const MetArgs &a, cudaStream_t st)
{
    const unsigned grid = (unsigned)((a.E + MET2_WARPS - 1) / MET2_WARPS);
    switch (L) {
#define HXG_MCASE(LL)                                                                                      \
    case LL:                                                                                               \
        metric_v2_kernel<S, LL><<<grid, MET2_WARPS * 32, 0, st>>>(a.E, a.kind, a.params, a.coef, a.wgrid, \
                                                                  a.tables, a.metric, a.status,           \
                                                                  a.status_or);                           \
        return cudaGetLastError() == cudaSuccess ? 0 : -5;
        HXG_MCASE(2) HXG_MCASE(3) HXG_MCASE(4) HXG_MCASE(5) HXG_MCASE(6)
        HXG_MCASE(7) HXG_MCASE(8) HXG_MCASE(9) HXG_MCASE(10) HXG_MCASE(11)
#undef HXG_MCASE
    }
    return 1;
}

// specialized extrusion-map kernel (simp_*_ext); returns 1 if none exists for p
template <int S>
int ext_launch(int p, const ExtArgs &a, cudaStream_t st)
{
    switch (p) {
#define HXG_CASE(PP) case PP: return launch_ext_t<S, PP>(a, st);
#ifndef HXG_QUICK_PS
        HXG_CASE(1) HXG_CASE(2) HXG_CASE(3) HXG_CASE(4) HXG_CASE(5)
        HXG_CASE(6) HXG_CASE(7) HXG_CASE(8) HXG_CASE(9) HXG_CASE(10)
#endif
#undef HXG_CASE
    }
    return 1;
}

}  // namespace hxg

// one translation unit per space: HXG_GEN_SPACE is the space code, HXG_GEN_NAME the
// suffix of the launcher names declared in hxg_v2_launch.h
#define HXG_GEN_CAT2(a, b) a##b
#define HXG_GEN_CAT(a, b) HXG_GEN_CAT2(a, b)
#define HXG_GEN_DEFINE_LAUNCHERS(SPACE, NAME)                                                             \
    namespace hxg {                                                                                     \
    int HXG_GEN_CAT(launch_v2_, NAME)(int p, const V2Args &a, cudaStream_t st) { return gen_launch<SPACE>(p, a, st); } \
    int HXG_GEN_CAT(launch_aff_, NAME)(int p, const AffV2Args &a, cudaStream_t st) { return aff_launch<SPACE>(p, a, st); } \
    int HXG_GEN_CAT(launch_ext_, NAME)(int p, const ExtArgs &a, cudaStream_t st) { return ext_launch<SPACE>(p, a, st); } \
    int HXG_GEN_CAT(launch_met_, NAME)(int L, const MetArgs &a, cudaStream_t st) { return met_launch<SPACE>(L, a, st); } \
    }
