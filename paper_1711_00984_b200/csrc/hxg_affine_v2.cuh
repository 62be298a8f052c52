// hxg_affine_v2.cuh -- compile-time specialized constant-Jacobian (affine) Gram
// kernel: simp_*_const of the reference (_kernels.py:1169-1404).
//
// With constant J every 1D integral is a closed-form F-table entry, so
//   G[J, I] = sum_h F_h[i1 + sa][j1 + sb] * Bs_h[a, i2, i3]     (<= 4 FMAs per entry)
//   Bs_h    = sum_{g in h} F_g[i2][j2] * sum_{t in g} sign * field_t * F_t[i3][j3]
// and the kernel is bound by the packed-output write.  One CTA owns the n1b
// packed rows J = (j1, j2, j3, b): the Bs sums go to shared memory, then each
// warp streams whole packed rows to HBM with coalesced stores (aff_rows).
#pragma once
#include <cstdlib>
#include "hxg_common.cuh"
#include "hxg_device.h"
#include "hxg_general_v2.cuh"
#include "hxg_geom.cuh"
#include "hxg_terms.h"

namespace hxg {

constexpr int AFF2_THREADS = 128;
#ifndef HXG_AFF_FLAT
#define HXG_AFF_FLAT 0  // 1: aff_rows deals (row, column chunk) items to the warps (measured 20-40 % slower: a warp streaming one contiguous row writes faster than warps interleaving chunks)
#endif

struct AffV2Args {
    const int *kind;
    const double *params, *coef, *tables;
    double *out;
    int *status;
    long long P;
    int E;
    int rg;  // row groups per CTA (aff_row_groups)
};

// Row groups per CTA: about 128 KB of output per CTA (per-CTA setup and tail
// effects dominate tiny row groups; whole elements for small elements), one
// group per CTA once a group alone carries >= 32 KB, and at least ~16 CTAs per
// SM.  Measured (profiles/affine_rg_r01.txt) on H1 p3-p10, H(curl) p4-p10,
// H(div) p5/p7.
inline int aff_row_groups(int NU, long long P, int E)
{
    long long target = 128LL << 10;
    if (const char *t = getenv("HXG_AFF_TARGET_KB")) target = 1024LL * atoll(t);  // tuning
    const double per_group = 8.0 * (double)P / NU;  // mean output bytes of one row group
    long long rg = per_group >= 32768.0 ? 1 : (long long)(target / per_group);
    rg = rg < 1 ? 1 : (rg > NU ? NU : rg);
    while (rg > 1 && (long long)E * ((NU + rg - 1) / rg) < (long long)sm_count() * 16) rg = (rg + 1) / 2;
    if (const char *r = getenv("HXG_AFF_RG")) rg = atoi(r) < 1 ? 1 : (atoi(r) > NU ? NU : atoi(r));  // tuning
    return (int)rg;
}

template <int S, int P>
struct AffCfg {
    static constexpr int NB = nb_of(S);
    __host__ __device__ static constexpr int n(int a, int d) { return ext_of(S, P, a, d); }
    __host__ __device__ static constexpr int blk(int a) { return n(a, 0) * n(a, 1) * n(a, 2); }
    __host__ __device__ static constexpr int off(int a)
    {
        return a == 0 ? 0 : (a == 1 ? blk(0) : blk(0) + blk(1));
    }
    static constexpr int N = off(NB - 1) + blk(NB - 1);
    __host__ __device__ static constexpr int nmax(int d)
    {
        return cmax(n(0, d), NB > 1 ? cmax(n(1, d), n(2, d)) : 0);
    }
    static constexpr int N1 = nmax(0);
    static constexpr int NK = cmax(n(0, 1) * n(0, 2), NB > 1 ? cmax(n(1, 1) * n(1, 2), n(2, 1) * n(2, 2)) : 0);
    static constexpr int BMAX = cmax(blk(0), NB > 1 ? cmax(blk(1), blk(2)) : 0);
    static constexpr int KF = P + 2;                 // F-table index range needed
    static constexpr int OFF_F = 0;                  // [4][KF][KF]
    static constexpr int OFF_B = OFF_F + 4 * KF * KF;  // [NB][NK][4]
    static constexpr int SMEM_BYTES = (OFF_B + NB * NK * 4) * 8;
    __host__ __device__ static constexpr int units()
    {
        int u = 0;
        for (int b = 0; b < NB; ++b) u += n(b, 1) * n(b, 2);
        return u;
    }
    static constexpr int NU = units();

};

// Direct variant: warp w writes packed rows j1 = w, w + 4, ...; lane (kq, i1) keeps its
// test digit i1 (and hence its F factors) fixed and walks column groups K with stride
// KW = 32 / n1a, so each warp store covers KW * n1a consecutive doubles of the row.
template <int S, int P, int A, int B>
__device__ __forceinline__ void aff_rows(const double *smem, double *__restrict__ outE, int j2, int j3,
                                         int bs_off = 0)  // bs_off: doubles past OFF_B (extrusion j2 slots)
{
    using C = AffCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int KF = C::KF, N = C::N;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n3a = C::n(A, 2);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha0 = sh_of(S, A, 0), shb0 = sh_of(S, B, 0);
    constexpr int offA = C::off(A), offB = C::off(B);
    constexpr int KW = n1a <= 32 ? 32 / n1a : 1;
    const double *sF = smem + C::OFF_F;
    const double *sBs = smem + C::OFF_B + bs_off + A * C::NK * 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane / n1a, i1 = lane - kq * n1a;
    const bool act = kq < KW;
    const int Kp = j2 + n2b * j3;
    const int K0 = (A == B) ? Kp : 0;
#if HXG_AFF_FLAT
    // (trial row j1, chunk of KW test columns K) items dealt round-robin to the warps: the
    // rows of a group are n1b = 5..11, which does not divide over the CTA's warps (a row
    // per warp left 1 of 4 warps busy in the last round at n1b = 9)
    constexpr int NW = AFF2_THREADS / 32;
    const int nch = (n2a * n3a - K0 + KW - 1) / KW;  // chunks per row (the same for every j1 of the group)
    int j1 = 0, ch = warp;
    while (ch >= nch) { ch -= nch; ++j1; }
    while (j1 < n1b) {
        double Fr[MAXH];
#pragma unroll
        for (int h = 0; h < MAXH; ++h)
            Fr[h] = h < pp.nh ? sF[((2 * pp.h_fr[h] + pp.h_fs[h]) * KF + i1 + sha0) * KF + j1 + shb0] : 0.0;
        const int J = offB + j1 + n1b * Kp;
        double *rowp = outE + (J * N - J * (J - 1) / 2 - J);  // &G(J, 0)
#pragma unroll 4
        for (; ch < nch; ch += NW) {
            const int K = K0 + kq + KW * ch;
            if (act && K < n2a * n3a) {
                const int I = offA + K * n1a + i1;
                const double2 b01 = *reinterpret_cast<const double2 *>(sBs + K * 4);
                double v = Fr[0] * b01.x;
                if (pp.nh > 1) v = fma(Fr[1], b01.y, v);
                if (pp.nh > 2) {
                    const double2 b23 = *reinterpret_cast<const double2 *>(sBs + K * 4 + 2);
                    v = fma(Fr[2], b23.x, v);
                    if (pp.nh > 3) v = fma(Fr[3], b23.y, v);
                }
                if (I >= J) __stcs(rowp + I, v);
            }
        }
        while (ch >= nch && j1 < n1b) { ch -= nch; ++j1; }
    }
#else
    for (int j1 = warp; j1 < n1b; j1 += AFF2_THREADS / 32) {
        double Fr[MAXH];
#pragma unroll
        for (int h = 0; h < MAXH; ++h)
            Fr[h] = h < pp.nh ? sF[((2 * pp.h_fr[h] + pp.h_fs[h]) * KF + i1 + sha0) * KF + j1 + shb0] : 0.0;
        const int J = offB + j1 + n1b * Kp;
        double *rowp = outE + (J * N - J * (J - 1) / 2 - J);  // &G(J, 0)
        if (act) {
#pragma unroll 4
            for (int K = K0 + kq; K < n2a * n3a; K += KW) {
                const int I = offA + K * n1a + i1;
                const double2 b01 = *reinterpret_cast<const double2 *>(sBs + K * 4);
                double v = Fr[0] * b01.x;
                if (pp.nh > 1) v = fma(Fr[1], b01.y, v);
                if (pp.nh > 2) {
                    const double2 b23 = *reinterpret_cast<const double2 *>(sBs + K * 4 + 2);
                    v = fma(Fr[2], b23.x, v);
                    if (pp.nh > 3) v = fma(Fr[3], b23.y, v);
                }
                if (I >= J) __stcs(rowp + I, v);
            }
        }
    }
#endif
}

// Bs_h[A][K] for one (test block A, trial block B) pair
template <int S, int P, int A, int B>
__device__ __forceinline__ void aff_bsum(double *smem, const double *s_field, int j2, int j3)
{
    using C = AffCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int KF = C::KF, n2a = C::n(A, 1), n3a = C::n(A, 2);
    constexpr int sa1 = sh_of(S, A, 1), sa2 = sh_of(S, A, 2), sb1 = sh_of(S, B, 1), sb2 = sh_of(S, B, 2);
    const double *sF = smem + C::OFF_F;
    for (int k = threadIdx.x; k < n2a * n3a; k += AFF2_THREADS) {
        const int i2 = k % n2a, i3 = k / n2a;
        double acc[MAXH] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            double sg = 0.0;
#pragma unroll
            for (int t = 0; t < pp.nt; ++t) {
                if (pp.t_g[t] != g) continue;
                const double f = sF[((2 * pp.t_fr[t] + pp.t_fs[t]) * KF + i3 + sa2) * KF + j3 + sb2];
                const double v = s_field[pp.t_field[t]] * f;
                sg += pp.t_sign[t] > 0 ? v : -v;
            }
            const double fb = sF[((2 * pp.g_fr[g] + pp.g_fs[g]) * KF + i2 + sa1) * KF + j2 + sb1];
            acc[pp.g_h[g]] = fma(fb, sg, acc[pp.g_h[g]]);
        }
        double2 *dst = reinterpret_cast<double2 *>(smem + C::OFF_B + (A * C::NK + k) * 4);
        dst[0] = make_double2(acc[0], acc[1]);
        dst[1] = make_double2(acc[2], acc[3]);
    }
}

template <int S, int P>
__global__ void __launch_bounds__(AFF2_THREADS) affine_v2_kernel(const __grid_constant__ AffV2Args args)
{
    using C = AffCfg<S, P>;
    constexpr int KF = C::KF;
    extern __shared__ __align__(16) double smem[];
    __shared__ double s_field[MAXF];
    const int tid = threadIdx.x;
    const int ncta = (C::NU + args.rg - 1) / args.rg;  // CTAs per element
    const int cta = blockIdx.x % ncta;
    const int e = blockIdx.x / ncta;
    double *sF = smem + C::OFF_F;
    for (int idx = tid; idx < 4 * KF * KF; idx += AFF2_THREADS) {
        const int rs = idx / (KF * KF), q = idx - rs * KF * KF, i = q / KF, j = q - i * KF;
        sF[idx] = args.tables[TAB_F + (rs * KT + i) * KT + j];
    }
    if (tid == 0) {
        double J[3][3], D[6], Cm[6];
        dev_jacobian(args.kind[e], args.params + 24LL * e, 0.5, 0.5, 0.5, J);
        const double det = dev_metrics(J, D, Cm);
        dev_fields(S, det, D, Cm, 1.0, args.coef ? args.coef[e] : 1.0, s_field);
        if (cta == 0)  // the element's whole status word (no zero-fill pass before the kernel)
            args.status[e] = (det > 0.0 ? 0 : 1) | (args.kind[e] > 2 ? 2 : 0);  // gram.py:170-174
    }
    double *__restrict__ outE = args.out + (long long)e * args.P;
    const int u1 = cmin(C::NU, (cta + 1) * args.rg);
    for (int u = cta * args.rg; u < u1; ++u) {
        int rem = u, b = 0;
#pragma unroll
        for (int bb = 0; bb < C::NB - 1; ++bb)
            if (b == bb && rem >= C::n(bb, 1) * C::n(bb, 2)) { rem -= C::n(bb, 1) * C::n(bb, 2); b = bb + 1; }
        int n2b = C::n(0, 1);
#pragma unroll
        for (int bb = 1; bb < C::NB; ++bb)
            if (b == bb) n2b = C::n(bb, 1);
        const int j2 = rem % n2b, j3 = rem / n2b;
        __syncthreads();  // fields / F ready; previous row group done with the Bs sums
        // Bs_h[a][K = (i2, i3)] for every test block a >= b
        if constexpr (C::NB == 1) {
            aff_bsum<S, P, 0, 0>(smem, s_field, j2, j3);
        } else {
            if (b == 0) {
                aff_bsum<S, P, 0, 0>(smem, s_field, j2, j3);
                aff_bsum<S, P, 1, 0>(smem, s_field, j2, j3);
                aff_bsum<S, P, 2, 0>(smem, s_field, j2, j3);
            } else if (b == 1) {
                aff_bsum<S, P, 1, 1>(smem, s_field, j2, j3);
                aff_bsum<S, P, 2, 1>(smem, s_field, j2, j3);
            } else {
                aff_bsum<S, P, 2, 2>(smem, s_field, j2, j3);
            }
        }
        __syncthreads();
        if constexpr (C::NB == 1) {
            aff_rows<S, P, 0, 0>(smem, outE, j2, j3);
        } else {
            if (b == 0) {
                aff_rows<S, P, 0, 0>(smem, outE, j2, j3);
                aff_rows<S, P, 1, 0>(smem, outE, j2, j3);
                aff_rows<S, P, 2, 0>(smem, outE, j2, j3);
            } else if (b == 1) {
                aff_rows<S, P, 1, 1>(smem, outE, j2, j3);
                aff_rows<S, P, 2, 1>(smem, outE, j2, j3);
            } else {
                aff_rows<S, P, 2, 2>(smem, outE, j2, j3);
            }
        }
    }
}

}  // namespace hxg