// hxg_general_lo.cuh -- general-map Gram kernel for low isotropic orders (p = 2..4,
// rule L = p + 1): whole slabs of packed rows per CTA, one work item per thread.
//
// Reference loops: tens_{h1,hcurl,hdiv,l2}_alt (_kernels.py:356-1150); the term /
// group model is hxg_plan.h.
//
// At these orders an element matrix is 3-360 KB and a (trial block b, digit j3) slab
// of packed rows -- one contiguous range of the packed upper triangle -- is at most
// 48 KB.  The warp-per-unit kernels (v3 / PW) spend their time on per-unit set-up and
// on short bulk copies there (5-29 % of the roofline).  This kernel keeps the element
// in one CTA instead:
//   fields   the metric fields of the element's L^3 points, evaluated in the kernel
//   per slab (b, j3):
//     stage A  Abar_g[a][i3][l][m] = sum_{t in g} sign_t sum_n M_t[n][l][m] u(i3,n) u(j3,n)
//              for every test block a >= b, in shared memory
//     stage BC one thread per item (a, i3, i2, j2): B_h[l] = sum_{g in h} sum_m
//              u(i2,m) u(j2,m) Abar_g[l][m] stays in registers (nh L doubles); the
//              thread then forms its n1b x n1a entries D = sum_{h,l} B_h[l] U_h[j1][i1][l]
//              (U = u_s(j1,l) u_r(i1,l), tabulated once per CTA, broadcast loads) and
//              drops them into the slab image in shared memory
//     write    the slab image is one contiguous piece of the packed output: coalesced
//              streaming stores by the whole CTA
// EB elements share a CTA pass (TPE = THREADS / EB threads each) so that the items of
// a slab fill the CTA at p = 2, 3.  Two CTA barriers per slab.
#pragma once
#include "hxg_common.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_geom.cuh"
#include "hxg_terms.h"

namespace hxg {

#ifndef HXG_LO_THREADS
#define HXG_LO_THREADS 256
#endif
constexpr int LO_THREADS = HXG_LO_THREADS;

template <int S, int P>
struct LoCfg {
    static constexpr int L = P + 1, L2Q = L * L, L3 = L * L * L;
    static constexpr int NB = nb_of(S), NF = nf_of(S);
    __host__ __device__ static constexpr int n(int a, int d) { return ext_of(S, P, a, d); }
    __host__ __device__ static constexpr int blk(int a) { return n(a, 0) * n(a, 1) * n(a, 2); }
    __host__ __device__ static constexpr int off(int a) { return a == 0 ? 0 : (a == 1 ? blk(0) : blk(0) + blk(1)); }
    static constexpr int N = off(NB - 1) + blk(NB - 1);
    static constexpr int LP = (L + 1) & ~1;      // 1D table row stride in shared memory (even: 16-byte loads)
    static constexpr int L2P = (L * L + 1) & ~1;  // Abar[g][i3] vector stride (even)
    // U tables: [pair][h][j1][i1][L], pairs in (b, a >= b) order
    // (rows [h][j1] of n1a * L doubles, padded to an even count)
    __host__ __device__ static constexpr int urow(int a) { return (n(a, 0) * L + 1) & ~1; }
    __host__ __device__ static constexpr int usz(int a, int b) { return make_pair_plan(S, a, b).nh * n(b, 0) * urow(a); }
    __host__ __device__ static constexpr int uoff(int a, int b)
    {
        int o = 0;
        for (int bb = 0; bb < NB; ++bb)
            for (int aa = bb; aa < NB; ++aa) {
                if (aa == a && bb == b) return o;
                o += usz(aa, bb);
            }
        return o;
    }
    static constexpr int U_TOT = uoff(NB, NB);  // no match: total
    // Abar of one slab: [a >= b][g][i3][L^2]
    __host__ __device__ static constexpr int asz(int a, int b) { return make_pair_plan(S, a, b).ng * n(a, 2) * L2P; }
    __host__ __device__ static constexpr int aoff(int a, int b)
    {
        int o = 0;
        for (int aa = b; aa < a; ++aa) o += asz(aa, b);
        return o;
    }
    __host__ __device__ static constexpr int amax()
    {
        int m = 0;
        for (int b = 0; b < NB; ++b) m = cmax(m, aoff(NB, b));
        return m;
    }
    static constexpr int A_TOT = amax();
    // slab image: rows J0 .. J0 + R - 1 of the packed triangle, R = n1b n2b
    __host__ __device__ static constexpr int imgmax()
    {
        int m = 0;
        for (int b = 0; b < NB; ++b) {
            const int R = n(b, 0) * n(b, 1), J0 = off(b);
            m = cmax(m, R * N - (R * J0 + R * (R - 1) / 2));
        }
        return m;
    }
    static constexpr int IMG = (imgmax() + 1) & ~1;
    // items of a slab: (a, i3, i2, j2)
    __host__ __device__ static constexpr int items(int b)
    {
        int m = 0;
        for (int a = b; a < NB; ++a) m += n(a, 2) * n(a, 1) * n(b, 1);
        return m;
    }
    __host__ __device__ static constexpr int itemsmax()
    {
        int m = 0;
        for (int b = 0; b < NB; ++b) m = cmax(m, items(b));
        return m;
    }
    static constexpr int SLOT = ((NF * L3 + 1) & ~1) + A_TOT + IMG;  // doubles per element slot (parts even)
    static constexpr int COMMON = 2 * KT * LP + U_TOT;
    // elements per CTA pass: fill the CTA with slab items, within ~100 KB
    __host__ __device__ static constexpr int pick_eb()
    {
        int eb = 1;
        for (int q = 2; q <= 8; q *= 2)
            if (q * itemsmax() <= LO_THREADS + LO_THREADS / 4 && (COMMON + q * SLOT) * 8 <= 100 * 1024) eb = q;
        return eb;
    }
    static constexpr int EB = pick_eb();
    static constexpr int TPE = LO_THREADS / EB;
    static constexpr int SMEM_BYTES = (COMMON + EB * SLOT) * 8;
    static constexpr bool OK = SMEM_BYTES <= 200 * 1024 && P >= 1 && P <= 5;
    static constexpr int MINB = cmax(1, cmin(2, (227 * 1024) / (SMEM_BYTES + 1024)));
};

template <int I>
struct PWIntLo {
    static constexpr int value = I;
};

struct LoArgs {
    const double *tables;
    double *out;
    long long P;
    int E;
    const int *kind;
    const double *params, *coef, *wgrid;
    int *status;
};

// stage A of one block pair for the slab (b, j3): Abar[g][i3][l*L+m] (vector stride L2P)
template <int S, int P, int A, int B>
__device__ __forceinline__ void lo_stage_a(const double *sT, const double *sM, double *sA, int j3, int tin)
{
    using C = LoCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int L = C::L, L2Q = C::L2Q, L3 = C::L3, LP = C::LP, L2P = C::L2P;
    constexpr int n3a = C::n(A, 2);
    constexpr int sha2 = sh_of(S, A, 2), shb2 = sh_of(S, B, 2);
    double *dst = sA + C::aoff(A, B);
    for (int idx = tin; idx < n3a * L2Q; idx += C::TPE) {
        const int lm = idx % L2Q, i3 = idx / L2Q;
        // the 1D products of the (at most four) xi3 function-code pairs
        double w3[2][2][L];
#pragma unroll
        for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int fs = 0; fs < 2; ++fs)
#pragma unroll
                for (int nn = 0; nn < L; ++nn)
                    w3[fr][fs][nn] = sT[(fr * KT + i3 + sha2) * LP + nn] * sT[(fs * KT + j3 + shb2) * LP + nn];
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < pp.nt; ++t) {
                if (pp.t_g[t] != g) continue;  // compile-time after unrolling
                const double *mf = sM + pp.t_field[t] * L3 + lm;
                double s = 0.0;
#pragma unroll
                for (int nn = 0; nn < L; ++nn) s = fma(mf[nn * L2Q], w3[pp.t_fr[t]][pp.t_fs[t]][nn], s);
                acc += pp.t_sign[t] > 0 ? s : -s;
            }
            dst[(g * n3a + i3) * L2P + lm] = acc;
        }
    }
}

// stages B and C of one block pair: one item (i3, i2, j2) per thread pass
template <int S, int P, int A, int B>
__device__ __forceinline__ void lo_stage_bc(const double *sT, const double *sU, const double *sA, double *sImg,
                                            int j3, int it0, int stride, int &base)
{
    using C = LoCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int L = C::L, L2Q = C::L2Q, LP = C::LP, N = C::N;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n3a = C::n(A, 2);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha1 = sh_of(S, A, 1), shb1 = sh_of(S, B, 1);
    constexpr int offA = C::off(A), offB = C::off(B);
    constexpr int NIT = n3a * n2a * n2b;
    const double *U = sU + C::uoff(A, B);
    const double *Ab = sA + C::aoff(A, B);
    const int J0 = offB + n1b * n2b * j3;  // first packed row of the slab
    // items of this pair occupy [base, base + NIT) of the slab's item list
    int gfirst = it0;  // this thread's first item index >= base (items it0, it0 + stride, ...)
    if (gfirst < base) gfirst += ((base - gfirst + stride - 1) / stride) * stride;
    for (int it = gfirst - base; it < NIT; it += stride) {
        const int i2 = it % n2a, r = it / n2a, j2 = r % n2b, i3 = r / n2b;
        if (A == B && (i3 < j3 || (i3 == j3 && i2 < j2))) continue;  // wholly below the diagonal
        // ---- stage B: B_h[l] in registers
        double Bh[pp.nh][L];
#pragma unroll
        for (int h = 0; h < pp.nh; ++h)
#pragma unroll
            for (int l = 0; l < L; ++l) Bh[h][l] = 0.0;
        // this item's xi2 1D values, both function codes (16-byte loads of even-stride rows)
        double ti[2][LP], tj[2][LP];
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int m = 0; m < LP; m += 2) {
                const double2 va = *reinterpret_cast<const double2 *>(sT + (f * KT + i2 + sha1) * LP + m);
                const double2 vb = *reinterpret_cast<const double2 *>(sT + (f * KT + j2 + shb1) * LP + m);
                ti[f][m] = va.x;
                ti[f][m + 1] = va.y;
                tj[f][m] = vb.x;
                tj[f][m + 1] = vb.y;
            }
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            double w[L];
#pragma unroll
            for (int m = 0; m < L; ++m) w[m] = ti[pp.g_fr[g]][m] * tj[pp.g_fs[g]][m];
            // Abar_g[i3] as a flat vector of L^2 (padded even) doubles: broadcast 16-byte loads
            const double2 *ag = reinterpret_cast<const double2 *>(Ab + (g * n3a + i3) * C::L2P);
            double av[C::L2P];
#pragma unroll
            for (int k = 0; k < C::L2P; k += 2) {
                const double2 v = ag[k / 2];
                av[k] = v.x;
                av[k + 1] = v.y;
            }
#pragma unroll
            for (int l = 0; l < L; ++l) {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < L; ++m) s = fma(w[m], av[l * L + m], s);
                Bh[pp.g_h[g]][l] += s;
            }
        }
        // ---- stage C: D[j1][i1] = sum_{h,l} B_h[l] U_h[j1][i1][l] into the slab image
        const int Ib = offA + n1a * (i2 + n2a * i3);
        constexpr int UR = C::urow(A);
#pragma unroll 1
        for (int j1 = 0; j1 < n1b; ++j1) {
            const int J = offB + j1 + n1b * (j2 + n2b * j3);
            // image offset of (J, J): rows J0 .. J - 1 hold N - J' entries each
            const int ro = (J - J0) * N - (J * (J - 1) / 2 - J0 * (J0 - 1) / 2) - J;
            double v[n1a];
#pragma unroll
            for (int i1 = 0; i1 < n1a; ++i1) v[i1] = 0.0;
#pragma unroll
            for (int h = 0; h < pp.nh; ++h) {
                const double2 *u2 = reinterpret_cast<const double2 *>(U + (h * n1b + j1) * UR);
                double uv[UR];
#pragma unroll
                for (int k = 0; k < UR; k += 2) {
                    const double2 x = u2[k / 2];
                    uv[k] = x.x;
                    uv[k + 1] = x.y;
                }
#pragma unroll
                for (int i1 = 0; i1 < n1a; ++i1)
#pragma unroll
                    for (int l = 0; l < L; ++l) v[i1] = fma(Bh[h][l], uv[i1 * L + l], v[i1]);
            }
#pragma unroll
            for (int i1 = 0; i1 < n1a; ++i1) {
                const int I = Ib + i1;
                if (A != B || I >= J) sImg[ro + I] = v[i1];
            }
        }
    }
    base += NIT;
}

template <int S, int P, int B>
__device__ __forceinline__ void lo_slab(const double *sT, const double *sU, const double *sM, double *sA,
                                        double *sImg, double *__restrict__ outE, int j3, int tin, bool live)
{
    using C = LoCfg<S, P>;
    constexpr int N = C::N;
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1), offB = C::off(B);
    if (live) {
        lo_stage_a<S, P, B, B>(sT, sM, sA, j3, tin);
        if constexpr (C::NB > 1 && B <= 1) lo_stage_a<S, P, B + 1 < 3 ? B + 1 : 2, B>(sT, sM, sA, j3, tin);
        if constexpr (C::NB > 1 && B == 0) lo_stage_a<S, P, 2, B>(sT, sM, sA, j3, tin);
    }
    __syncthreads();  // Abar ready; the previous slab's image has been written out
    if (live) {
        int base = 0;
        lo_stage_bc<S, P, B, B>(sT, sU, sA, sImg, j3, tin, C::TPE, base);
        if constexpr (C::NB > 1 && B <= 1) lo_stage_bc<S, P, B + 1 < 3 ? B + 1 : 2, B>(sT, sU, sA, sImg, j3, tin, C::TPE, base);
        if constexpr (C::NB > 1 && B == 0) lo_stage_bc<S, P, 2, B>(sT, sU, sA, sImg, j3, tin, C::TPE, base);
    }
    __syncthreads();  // image complete
    if (live) {
        constexpr int R = n1b * n2b;
        const int J0 = offB + R * j3;
        const int len = R * N - (R * J0 + R * (R - 1) / 2);
        double *dst = outE + ((long long)J0 * N - (long long)J0 * (J0 - 1) / 2);
        for (int k = tin; k < len; k += C::TPE) __stcs(dst + k, sImg[k]);
    }
}

template <int S, int P>
__global__ void __launch_bounds__(LO_THREADS, (LoCfg<S, P>::MINB)) general_lo_kernel(const __grid_constant__ LoArgs args)
{
    using C = LoCfg<S, P>;
    constexpr int L = C::L, L3 = C::L3, LP = C::LP, NB = C::NB;
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x;
    double *sT = smem;                 // [2][KT][LP]
    double *sU = smem + 2 * KT * LP;   // U tables of every block pair
    for (int idx = tid; idx < 2 * KT * LP; idx += LO_THREADS) {
        const int fk = idx / LP, l = idx - fk * LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    __syncthreads();
    // U_h[j1][i1][l] = u_s(j1, l) u_r(i1, l) for every pair (b, a >= b)
    auto fill_u = [&](auto ac, auto bc) {
        constexpr int A = decltype(ac)::value, B = decltype(bc)::value;
        constexpr CPair pp = make_pair_plan(S, A, B);
        constexpr int n1a = C::n(A, 0), n1b = C::n(B, 0);
        constexpr int sha0 = sh_of(S, A, 0), shb0 = sh_of(S, B, 0);
        double *U = sU + C::uoff(A, B);
        constexpr int UR = C::urow(A);
        for (int idx = tid; idx < pp.nh * n1b * UR; idx += LO_THREADS) {
            const int k = idx % UR, r2 = idx / UR, j1 = r2 % n1b, h = r2 / n1b;
            const int i1 = k / L, l = k - i1 * L;
            int fr = 0, fs = 0;
#pragma unroll
            for (int hh = 0; hh < pp.nh; ++hh)
                if (hh == h) { fr = pp.h_fr[hh]; fs = pp.h_fs[hh]; }
            U[idx] = i1 < n1a ? sT[(fs * KT + j1 + shb0) * LP + l] * sT[(fr * KT + i1 + sha0) * LP + l] : 0.0;
        }
    };
    fill_u(PWIntLo<0>{}, PWIntLo<0>{});
    if constexpr (NB > 1) {
        fill_u(PWIntLo<1>{}, PWIntLo<0>{});
        fill_u(PWIntLo<2>{}, PWIntLo<0>{});
        fill_u(PWIntLo<1>{}, PWIntLo<1>{});
        fill_u(PWIntLo<2>{}, PWIntLo<1>{});
        fill_u(PWIntLo<2>{}, PWIntLo<2>{});
    }
    const int slot = tid / C::TPE, tin = tid - slot * C::TPE;
    double *sM = smem + C::COMMON + slot * C::SLOT;  // [NF][L3]
    double *sA = sM + ((C::NF * L3 + 1) & ~1);
    double *sImg = sA + C::A_TOT;
    for (long long e0 = (long long)blockIdx.x * C::EB; e0 < args.E; e0 += (long long)gridDim.x * C::EB) {
        const long long e = e0 + slot;
        const bool live = e < args.E;
        __syncthreads();  // U tables (first pass); previous pass done with sM
        if (live) {
            const double *par = args.params + 24LL * e;
            const int knd = args.kind[e];
            const double cf = args.coef ? args.coef[e] : 1.0;
            for (int pt = tin; pt < L3; pt += C::TPE) {
                const int nn = pt / (L * L), l = (pt / L) % L, m = pt % L;
                double J[3][3], D[6], Cm[6], f[MAXF];
                dev_jacobian(knd, par, args.tables[TAB_NODES + l], args.tables[TAB_NODES + m],
                             args.tables[TAB_NODES + nn], J);
                const double det = dev_metrics(J, D, Cm);
                const double w = args.tables[TAB_WTS + l] * args.tables[TAB_WTS + m] * args.tables[TAB_WTS + nn];
                const double c = args.wgrid ? args.wgrid[e * L3 + (l * L + m) * L + nn] : cf;
                dev_fields(S, det, D, Cm, w, c, f);
#pragma unroll
                for (int k = 0; k < C::NF; ++k) sM[k * L3 + pt] = f[k];
                if (!(det > 0.0)) atomicOr(args.status + e, 1);
            }
        }
        __syncthreads();
        double *__restrict__ outE = args.out + (live ? e : 0) * args.P;
        for (int j3 = 0; j3 < C::n(0, 2); ++j3) lo_slab<S, P, 0>(sT, sU, sM, sA, sImg, outE, j3, tin, live);
        if constexpr (NB > 1) {
            for (int j3 = 0; j3 < C::n(1, 2); ++j3) lo_slab<S, P, 1>(sT, sU, sM, sA, sImg, outE, j3, tin, live);
            for (int j3 = 0; j3 < C::n(2, 2); ++j3) lo_slab<S, P, 2>(sT, sU, sM, sA, sImg, outE, j3, tin, live);
        }
    }
}

}  // namespace hxg
