// hxg_extrusion.cuh -- simplified Gram path for extrusion maps (O(p^6)).
//
// Reference: gram.py:192-203 -> simp_{l2,h1,hdiv,hcurl}_ext (_kernels.py:1405-1764).
// An extrusion map (kind 3, geometry.py:100-111) is affine in xi1 alone and a
// planar bilinear quad in (xi2, xi3), so its Jacobian is block diagonal and
// independent of xi1: the xi1 integrals are the closed-form F tables (as on the
// constant-Jacobian path) and only (xi2, xi3) needs quadrature, on the L x L
// grid at xi1 = 0.5.
//
// Work unit: a slab (element, trial block b, digit j3) -- all packed row groups
// j2 of the slab; rg slabs per CTA (aff_row_groups at slab granularity):
//   stage A  Abar_g[a][i3][m] = sum_{t in g} sign_t sum_n M_t[m][n] u(i3,n) u(j3,n)
//            (once per slab, for every test block a >= b)
//   per pass of jc trial digits j2 (shared-memory budget):
//   stage B  Bs_h[a][(i2,i3)] = sum_{g in h} sum_m u(i2,m) u(j2,m) Abar_g[a][i3][m]
//   rows     G[J][I] = sum_h F_h[i1][j1] Bs_h[(i2,i3)]        (aff_rows, shared)
// with the per-point term fields M_t (w_m w_n folded in, hxg_geom.cuh) evaluated
// once per CTA in shared memory.  The output stream dominates: HBM-write bound.
#pragma once
#include <algorithm>
#include "hxg_affine_v2.cuh"

namespace hxg {

struct ExtArgs {
    const int *kind;
    const double *params, *coef, *tables;
    double *out;
    int *status;
    long long P;
    int E;
    int rg;  // row groups per CTA (aff_row_groups)
    int L;   // rule order in xi2 and xi3 (gram.py:192-195)
    int jc;  // trial digits j2 whose Bs sums are built per pass (host: smem budget)
};

#ifndef HXG_EXT_VT
#define HXG_EXT_VT 1
#endif

template <int S, int P>
struct ExtCfg {
    using A = AffCfg<S, P>;
    static constexpr int NB = A::NB, NK = A::NK, NU = A::NU;
    __host__ __device__ static constexpr int n(int a, int d) { return A::n(a, d); }
    __host__ __device__ static constexpr int maxg()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b < NB; ++b) m = cmax(m, make_pair_plan(S, a, b).ng);
        return m;
    }
    static constexpr int NG = maxg();
    static constexpr int N3 = A::nmax(2);
    static constexpr int NF = nf_of(S);
    // shared memory (doubles): [F tables | Bs] of AffCfg, then the 1D tables at the
    // rule nodes, the term fields and Abar; the last two scale with the runtime L
    static constexpr int OFF_T = A::SMEM_BYTES / 8;
    static constexpr int OFF_M = OFF_T + 2 * KT * LT;
    __host__ __device__ static constexpr int off_abar(int L) { return OFF_M + NF * L * L; }
    __host__ __device__ static constexpr int off_bs(int L) { return (off_abar(L) + NB * N3 * NG * L + 1) & ~1; }  // double2
    static constexpr int BS_SLOT = NB * NK * 4;  // Bs of one j2, every test block
    // stage-B factor table Vt[jj][fr 2 + fs][ra][m] = u_fr(ra, m) u_fs(j2 + sb1, m) of the
    // current j2 chunk (HXG_EXT_VT): formed once per chunk instead of per (i2, i3, g) item
    static constexpr int KF = A::KF;
    // stage-B digits i3 per thread item (see ext_stage_b); the Vt table serves C3 == 1
#ifdef HXG_EXT_C3
    static constexpr int C3 = HXG_EXT_C3;
#else
    // (H1 p = 7, n3 = 8: C3 = 2 measured 29 -> 49 % of the roofline; at every other H1 order
    // C3 = 2 / 4 measured slower, 22-50 % vs 25-65 %)
    static constexpr int C3 = (S == HDIV && P >= 6) ? 4 : ((S == H1 && P == 7) ? 2 : 1);
#endif
    static constexpr bool VT = HXG_EXT_VT && C3 == 1;
    __host__ __device__ static constexpr int vt_slot(int L) { return VT ? 4 * KF * L : 0; }
    __host__ __device__ static constexpr int off_vt(int L, int jc) { return off_bs(L) + jc * BS_SLOT; }
    __host__ __device__ static constexpr int smem_bytes(int L, int jc)
    {
        return (off_vt(L, jc) + jc * vt_slot(L)) * 8;
    }
};

template <int I>
struct ExtInt {
    static constexpr int value = I;
};

// stage A for test block A of the (A, B) pair: Abar[A][i3][g][m]
// (LC: the rule order as a compile-time constant, 0 = runtime L)
template <int S, int P, int LC, int A, int B>
__device__ __forceinline__ void ext_stage_a(double *smem, int Lr, int j3)
{
    const int L = LC ? LC : Lr;
    using C = ExtCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int n3a = C::n(A, 2), NG = C::NG, N3 = C::N3;
    constexpr int sa2 = sh_of(S, A, 2), sb2 = sh_of(S, B, 2);
    const double *sT = smem + C::OFF_T, *sM = smem + C::OFF_M;
    double *sAb = smem + C::off_abar(L) + (size_t)A * N3 * NG * L;
    const int LL = L * L;
    if constexpr (LC >= 1 && LC <= 8) {
    // a thread owns (i3, m) and every GC-th term group; groups and terms are compile-time
    // (with a runtime group index every thread ran all nt terms predicated: 17 % of the
    // H1 p6 kernel's warp samples)
    constexpr int GC = pp.ng >= 6 ? 3 : (pp.ng >= 2 ? 2 : 1);
    for (int idx = threadIdx.x; idx < n3a * L * GC; idx += AFF2_THREADS) {
        const int m = idx % L, q = idx / L, i3 = q % n3a, c = q / n3a;
        // xi3 1D products of the four function-code pairs
        double w3[2][2][LC ? LC : LT];
#pragma unroll
        for (int fr = 0; fr < 2; ++fr)
#pragma unroll
            for (int fs = 0; fs < 2; ++fs)
#pragma unroll
                for (int nn = 0; nn < (LC ? LC : LT); ++nn)
                    w3[fr][fs][nn] = (LC || nn < L) ? sT[(fr * KT + i3 + sa2) * LT + nn] * sT[(fs * KT + j3 + sb2) * LT + nn] : 0.0;
        auto run = [&](auto cc) {
            constexpr int CC = decltype(cc)::value;
            constexpr CPair pq = make_pair_plan(S, A, B);  // not captured: stays a compile-time constant
#pragma unroll
            for (int g = 0; g < pq.ng; ++g) {
                if (g % GC != CC) continue;
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < pq.nt; ++t) {
                    if (pq.t_g[t] != g) continue;
                    const double *Mt = sM + pq.t_field[t] * LL + m * L;
                    double s = 0.0;
#pragma unroll
                    for (int nn = 0; nn < (LC ? LC : LT); ++nn)
                        if (LC || nn < L) s = fma(Mt[nn], w3[pq.t_fr[t]][pq.t_fs[t]][nn], s);
                    acc += pq.t_sign[t] > 0 ? s : -s;
                }
                sAb[(i3 * NG + g) * L + m] = acc;
            }
        };
        if (c == 0) run(ExtInt<0>{});
        if constexpr (GC > 1) if (c == 1) run(ExtInt<1>{});
        if constexpr (GC > 2) if (c == 2) run(ExtInt<2>{});
    }
    } else {
    // long rules (L > 8: the four 1D product vectors would cost more registers than they
    // save; measured -20 % at p = 10) and runtime L: one (i3, g, m) entry per thread
    for (int idx = threadIdx.x; idx < n3a * pp.ng * L; idx += AFF2_THREADS) {
        const int m = idx % L, q = idx / L, g = q % pp.ng, i3 = q / pp.ng;
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < pp.nt; ++t) {
            if (pp.t_g[t] != g) continue;
            const double *Mt = sM + pp.t_field[t] * LL + m * L;
            const double *Ta = sT + (pp.t_fr[t] * KT + i3 + sa2) * LT;
            const double *Tb = sT + (pp.t_fs[t] * KT + j3 + sb2) * LT;
            double s = 0.0;
#pragma unroll
            for (int nn = 0; nn < (LC ? LC : LT); ++nn)
                if (LC || nn < L) s = fma(Mt[nn], Ta[nn] * Tb[nn], s);
            acc += pp.t_sign[t] > 0 ? s : -s;
        }
        sAb[(i3 * NG + g) * L + m] = acc;
    }
    }
}

// stage B for test block A of the (A, B) pair: Bs_h[A][k = i2 + n2a i3][h]
template <int S, int P, int LC, int A, int B>
__device__ __forceinline__ void ext_stage_b(double *smem, int Lr, int j2lo, int jn, int jc)
{
    using C = ExtCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int n2a = C::n(A, 1), n3a = C::n(A, 2), NG = C::NG, N3 = C::N3;
    constexpr int sa1 = sh_of(S, A, 1), sb1 = sh_of(S, B, 1);
    const int L = LC ? LC : Lr;
    const double *sT = smem + C::OFF_T;
    const double *sAb = smem + C::off_abar(L) + (size_t)A * N3 * NG * L;
    // a thread owns (j2, i2) and up to C3 digits i3: the factor u(i2, m) u(j2, m) of
    // each group is formed once and reused for its i3 digits (it does not depend on i3).
    // Measured (config-5 sweep): C3 = 4 lifts H(div) at p >= 6 (75-95 % vs 69-90 %) but
    // starves p <= 5 of thread items; H1 / H(curl) (up to 9 groups) lose occupancy to
    // the accumulators: C3 = 1 there.
    constexpr int C3 = C::C3;
    if constexpr (C3 == 1) {
    const double *sVt = smem + C::off_vt(L, jc);
    (void)sVt;
    for (int it = threadIdx.x; it < jn * n2a * n3a; it += AFF2_THREADS) {
        const int jj = it / (n2a * n3a), k = it - jj * (n2a * n3a), j2 = j2lo + jj;
        const int i2 = k % n2a, i3 = k / n2a;
        double acc[MAXH] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            const double *Ab = sAb + (i3 * NG + g) * L;
            double s = 0.0;
            if constexpr (C::VT) {
                const double *V = sVt + ((jj * 4 + pp.g_fr[g] * 2 + pp.g_fs[g]) * C::KF + i2 + sa1) * L;
#pragma unroll
                for (int m = 0; m < (LC ? LC : LT); ++m)
                    if (LC || m < L) s = fma(V[m], Ab[m], s);
            } else {
                const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sa1) * LT;
                const double *Tb = sT + (pp.g_fs[g] * KT + j2 + sb1) * LT;
#pragma unroll
                for (int m = 0; m < (LC ? LC : LT); ++m)
                    if (LC || m < L) s = fma(Ta[m] * Tb[m], Ab[m], s);
            }
            acc[pp.g_h[g]] += s;
        }
        double2 *dst = reinterpret_cast<double2 *>(smem + C::off_bs(L) + jj * C::BS_SLOT + (A * C::NK + k) * 4);
        dst[0] = make_double2(acc[0], acc[1]);
        dst[1] = make_double2(acc[2], acc[3]);
    }
    } else {
    constexpr int NCI = (n3a + C3 - 1) / C3;
    constexpr int LV = LC ? LC : LT;
    for (int it = threadIdx.x; it < jn * n2a * NCI; it += AFF2_THREADS) {
        const int jj = it / (n2a * NCI), r = it - jj * (n2a * NCI);
        const int ic = r / n2a, i2 = r - ic * n2a;  // consecutive threads: consecutive i2
        const int i3lo = ic * C3, j2 = j2lo + jj;
        double acc[C3][MAXH];
#pragma unroll
        for (int c = 0; c < C3; ++c)
#pragma unroll
            for (int h = 0; h < MAXH; ++h) acc[c][h] = 0.0;
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sa1) * LT;
            const double *Tb = sT + (pp.g_fs[g] * KT + j2 + sb1) * LT;
            double V[LV];
#pragma unroll
            for (int m = 0; m < LV; ++m) V[m] = (LC || m < L) ? Ta[m] * Tb[m] : 0.0;
#pragma unroll
            for (int c = 0; c < C3; ++c) {
                if (i3lo + c < n3a) {
                    const double *Ab = sAb + ((i3lo + c) * NG + g) * L;
                    double s = 0.0;
#pragma unroll
                    for (int m = 0; m < LV; ++m)
                        if (LC || m < L) s = fma(V[m], Ab[m], s);
                    acc[c][pp.g_h[g]] += s;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < C3; ++c) {
            if (i3lo + c < n3a) {
                const int k = i2 + n2a * (i3lo + c);
                double2 *dst = reinterpret_cast<double2 *>(smem + C::off_bs(L) + jj * C::BS_SLOT + (A * C::NK + k) * 4);
                dst[0] = make_double2(acc[c][0], acc[c][1]);
                dst[1] = make_double2(acc[c][2], acc[c][3]);
            }
        }
    }
    }
}

template <int S, int P>
__host__ __device__ constexpr int ext_slabs()
{
    return ExtCfg<S, P>::NB == 1 ? ExtCfg<S, P>::n(0, 2)
                                 : ExtCfg<S, P>::n(0, 2) + ExtCfg<S, P>::n(1, 2) + ExtCfg<S, P>::n(2, 2);
}

template <int S, int P, int LC>
__device__ __forceinline__ void ext_stage_a_all(double *smem, int L, int b, int j3)
{
    if constexpr (ExtCfg<S, P>::NB == 1) {
        ext_stage_a<S, P, LC, 0, 0>(smem, L, j3);
    } else if (b == 0) {
        ext_stage_a<S, P, LC, 0, 0>(smem, L, j3);
        ext_stage_a<S, P, LC, 1, 0>(smem, L, j3);
        ext_stage_a<S, P, LC, 2, 0>(smem, L, j3);
    } else if (b == 1) {
        ext_stage_a<S, P, LC, 1, 1>(smem, L, j3);
        ext_stage_a<S, P, LC, 2, 1>(smem, L, j3);
    } else {
        ext_stage_a<S, P, LC, 2, 2>(smem, L, j3);
    }
}

template <int S, int P, int LC>
__device__ __forceinline__ void ext_stage_b_all(double *smem, int L, int b, int j2lo, int jn, int jc)
{
    if constexpr (ExtCfg<S, P>::NB == 1) {
        ext_stage_b<S, P, LC, 0, 0>(smem, L, j2lo, jn, jc);
    } else if (b == 0) {
        ext_stage_b<S, P, LC, 0, 0>(smem, L, j2lo, jn, jc);
        ext_stage_b<S, P, LC, 1, 0>(smem, L, j2lo, jn, jc);
        ext_stage_b<S, P, LC, 2, 0>(smem, L, j2lo, jn, jc);
    } else if (b == 1) {
        ext_stage_b<S, P, LC, 1, 1>(smem, L, j2lo, jn, jc);
        ext_stage_b<S, P, LC, 2, 1>(smem, L, j2lo, jn, jc);
    } else {
        ext_stage_b<S, P, LC, 2, 2>(smem, L, j2lo, jn, jc);
    }
}

// Vt of the j2 chunk [j2lo, j2lo + jn) for trial block b (written while no one reads it)
template <int S, int P>
__device__ __forceinline__ void ext_build_vt(double *smem, int L, int b, int j2lo, int jn, int jc)
{
    using C = ExtCfg<S, P>;
    if constexpr (C::VT) {
        const double *sT = smem + C::OFF_T;
        double *sVt = smem + C::off_vt(L, jc);
        const int sb1 = sh_of(S, b, 1);
        for (int idx = threadIdx.x; idx < jn * 4 * C::KF * L; idx += AFF2_THREADS) {
            const int m = idx % L, q = idx / L, ra = q % C::KF, q2 = q / C::KF, combo = q2 & 3, jj = q2 >> 2;
            sVt[idx] = sT[((combo >> 1) * KT + ra) * LT + m] * sT[((combo & 1) * KT + j2lo + jj + sb1) * LT + m];
        }
    }
}

template <int S, int P>
__device__ __forceinline__ void ext_rows_all(const double *smem, double *outE, int b, int j2, int j3, int off)
{
    if constexpr (ExtCfg<S, P>::NB == 1) {
        aff_rows<S, P, 0, 0>(smem, outE, j2, j3, off);
    } else if (b == 0) {
        aff_rows<S, P, 0, 0>(smem, outE, j2, j3, off);
        aff_rows<S, P, 1, 0>(smem, outE, j2, j3, off);
        aff_rows<S, P, 2, 0>(smem, outE, j2, j3, off);
    } else if (b == 1) {
        aff_rows<S, P, 1, 1>(smem, outE, j2, j3, off);
        aff_rows<S, P, 2, 1>(smem, outE, j2, j3, off);
    } else {
        aff_rows<S, P, 2, 2>(smem, outE, j2, j3, off);
    }
}

template <int S, int P, int LC>
__global__ void __launch_bounds__(AFF2_THREADS) ext_v2_kernel(const __grid_constant__ ExtArgs args)
{
    using C = ExtCfg<S, P>;
    using CA = typename C::A;
    constexpr int KF = CA::KF, NS = ext_slabs<S, P>();
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, L = LC ? LC : args.L, LL = L * L;
    const int ncta = (NS + args.rg - 1) / args.rg;  // CTAs per element (rg slabs each)
    const int cta = blockIdx.x % ncta;
    const int e = blockIdx.x / ncta;
    double *sF = smem + CA::OFF_F, *sT = smem + C::OFF_T, *sM = smem + C::OFF_M;
    for (int idx = tid; idx < 4 * KF * KF; idx += AFF2_THREADS) {
        const int rs = idx / (KF * KF), q = idx - rs * KF * KF, i = q / KF, j = q - i * KF;
        sF[idx] = args.tables[TAB_F + (rs * KT + i) * KT + j];
    }
    for (int idx = tid; idx < 2 * KT * LT; idx += AFF2_THREADS) sT[idx] = args.tables[TAB_T + idx];
    // term fields on the (xi2, xi3) grid at xi1 = 0.5, weight w_m w_n
    // (_kernels.py:1429-1434, 1481-1494, 1568-1589, 1683-1711)
    {
        const int knd = args.kind[e];
        const double *par = args.params + 24LL * e;
        const double cf = args.coef ? args.coef[e] : 1.0;
        bool bad = false;
        for (int pt = tid; pt < LL; pt += AFF2_THREADS) {
            const int m = pt / L, nn = pt - m * L;
            double J[3][3], D[6], Cm[6], f[MAXF];
            dev_jacobian(knd, par, 0.5, args.tables[TAB_NODES + m], args.tables[TAB_NODES + nn], J);
            const double det = dev_metrics(J, D, Cm);
            dev_fields(S, det, D, Cm, args.tables[TAB_WTS + m] * args.tables[TAB_WTS + nn], cf, f);
#pragma unroll
            for (int k = 0; k < C::NF; ++k) sM[k * LL + pt] = f[k];
            bad |= !(det > 0.0);
        }
        if (cta == 0) {
            if (bad) atomicOr(args.status + e, 1);
            if (tid == 0 && knd > 3) atomicOr(args.status + e, 2);  // gram.py:170-174
        }
    }
    double *__restrict__ outE = args.out + (long long)e * args.P;
    const int s1 = cmin(NS, (cta + 1) * args.rg);
    for (int sl = cta * args.rg; sl < s1; ++sl) {
        int j3 = sl, b = 0;
#pragma unroll
        for (int bb = 0; bb < C::NB - 1; ++bb)
            if (b == bb && j3 >= C::n(bb, 2)) { j3 -= C::n(bb, 2); b = bb + 1; }
        int n2b = C::n(0, 1);
#pragma unroll
        for (int bb = 1; bb < C::NB; ++bb)
            if (b == bb) n2b = C::n(bb, 1);
        __syncthreads();  // fields ready; previous slab done with Abar / Bs / Vt
        ext_stage_a_all<S, P, LC>(smem, L, b, j3);
        ext_build_vt<S, P>(smem, L, b, 0, cmin(args.jc, n2b), args.jc);
        for (int j2lo = 0; j2lo < n2b; j2lo += args.jc) {
            const int jn = cmin(args.jc, n2b - j2lo);
            __syncthreads();  // Abar / Vt complete; previous rows done with the Bs slots
            ext_stage_b_all<S, P, LC>(smem, L, b, j2lo, jn, args.jc);
            __syncthreads();
            const int off = C::off_bs(L) - CA::OFF_B;  // aff_rows reads OFF_B + off + slot
            for (int jj = 0; jj < jn; ++jj)
                ext_rows_all<S, P>(smem, outE, b, j2lo + jj, j3, off + jj * C::BS_SLOT);
            if (j2lo + args.jc < n2b)  // stage B of this chunk is done with Vt
                ext_build_vt<S, P>(smem, L, b, j2lo + args.jc, cmin(args.jc, n2b - j2lo - args.jc), args.jc);
        }
    }
}

// host launcher for one (space, p); returns 0, 1 (no specialization) or < 0
template <int S, int P>
inline int launch_ext_t(const ExtArgs &a, cudaStream_t st)
{
    using C = ExtCfg<S, P>;
    constexpr int NS = ext_slabs<S, P>();
    // Bs of jc trial digits per pass (one barrier pair per pass instead of per j2)
    const int n2max = C::A::nmax(1);
    long long budget = 24LL * 1024;
    if (const char *t = getenv("HXG_EXT_SMEM_KB")) budget = 1024LL * atoll(t);  // tuning
    int jc = (int)std::min<long long>(
        n2max, std::max<long long>(1, (budget / 8 - C::off_bs(a.L)) / (C::BS_SLOT + C::vt_slot(a.L))));
    const size_t smem = C::smem_bytes(a.L, jc);
    if (smem > 200 * 1024) return 1;
    // the reference's default rule (L = p + 1) unrolls; other rules loop
    auto k = a.L == P + 1 ? ext_v2_kernel<S, P, P + 1> : ext_v2_kernel<S, P, 0>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -5;
    ExtArgs b = a;
    b.jc = jc;
    // slabs per CTA: ~128 KB of output per CTA, >= 16 CTAs per SM (aff_row_groups
    // on slab granularity)
    b.rg = aff_row_groups(NS, a.P, a.E);
    const long long grid = (long long)a.E * ((NS + b.rg - 1) / b.rg);
    if (grid >= (1ll << 31)) return -6;
    k<<<(int)grid, AFF2_THREADS, smem, st>>>(b);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

}  // namespace hxg
