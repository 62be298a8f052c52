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
#define HXG_LO_THREADS 128
#endif
constexpr int LO_THREADS = HXG_LO_THREADS;
#ifndef HXG_LO_BUDGET_KB
#define HXG_LO_BUDGET_KB 44  // shared memory per CTA (4 CTAs per SM: more barrier domains per SM measured +3-14 % over 2 x 256 threads)
#endif
#ifndef HXG_LO_MAXB
#define HXG_LO_MAXB 5  // CTAs per SM (5 x 128 threads at <= 102 registers: +2-6 % over 4) (register budget 65536 / (MAXB * THREADS))
#endif
#ifndef HXG_LO_J1U
#define HXG_LO_J1U 1  // unroll factor of the stage-C trial-row loop (2 measured -4 to -18 %)
#endif
#ifndef HXG_LO_EBMAX
#define HXG_LO_EBMAX 16  // most elements per CTA pass
#endif

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
    static constexpr int A_TOT1 = amax();  // Abar of one slab
    // image of nj consecutive slabs of a block: rows J0 .. J0 + nj R - 1 of the packed triangle
    __host__ __device__ static constexpr int imgmax(int nj)
    {
        int m = 0;
        for (int b = 0; b < NB; ++b) {
            const int R = n(b, 0) * n(b, 1) * cmin(nj, n(b, 2)), J0 = off(b);
            m = cmax(m, R * N - (R * J0 + R * (R - 1) / 2));
        }
        return (m + 1) & ~1;
    }
    __host__ __device__ static constexpr int n3max() { return cmax(n(0, 2), NB > 1 ? cmax(n(1, 2), n(2, 2)) : 0); }
    __host__ __device__ static constexpr int slot(int nj) { return ((NF * L3 + 1) & ~1) + nj * A_TOT1 + imgmax(nj); }
    static constexpr int COMMON = 2 * KT * LP + U_TOT;
    static constexpr int BUDGET = (HXG_LO_BUDGET_KB * 1024) / 8;  // doubles per CTA
    __host__ __device__ static constexpr int eb_of(int nj) { return cmin(HXG_LO_EBMAX, (BUDGET - COMMON) / slot(nj)); }
    // slabs per pass: the most (slabs x elements) in flight between two barriers
    __host__ __device__ static constexpr int pick_nj()
    {
        int best = 1, score = 0;
        for (int nj = 1; nj <= n3max(); ++nj) {
            // average slabs per pass (x 60, exact for n3 <= 5) times the elements of a pass
            const int passes = (n3max() + nj - 1) / nj;
            const int sc = eb_of(nj) * (60 * n3max() / passes);
            if (sc >= score && eb_of(nj) >= 1) { score = sc; best = nj; }
        }
        return best;
    }
    // single-block spaces (H1, L2): one slab per pass and as many elements as fill the CTA
    // with slab items (measured: H1 p3 60 vs 52 M el/s for whole-element passes -- idle
    // warps of a short slab cost nothing while the SM's other CTA runs)
    __host__ __device__ static constexpr int eb_single()
    {
        const int items = n(0, 2) * n(0, 1) * n(0, 1);
        int eb = 1;
        for (int q = 2; q <= HXG_LO_EBMAX; q *= 2)
            if (q * items <= LO_THREADS + LO_THREADS / 4 && q <= eb_of(1)) eb = q;
        return eb;
    }
    static constexpr int NJ3 = NB == 1 ? 1 : pick_nj();
    static constexpr int EB = NB == 1 ? eb_single() : cmax(1, eb_of(NJ3));
    static constexpr int A_TOT = NJ3 * A_TOT1;
    static constexpr int IMG = imgmax(NJ3);
    static constexpr int SLOT = slot(NJ3);  // doubles per element slot (parts even)
    static constexpr int TPE = LO_THREADS / EB;
    static constexpr int SMEM_BYTES = (COMMON + EB * SLOT) * 8;
    static constexpr bool OK = SMEM_BYTES <= 200 * 1024 && P >= 1 && P <= 5;
    static constexpr int MINB = cmax(1, cmin(HXG_LO_MAXB, (227 * 1024) / (SMEM_BYTES + 1024)));
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

// stages B and C of one item (i3, i2, j2) of block pair (A, B) in the slab (b, j3)
template <int S, int P, int A, int B>
__device__ __forceinline__ void lo_item(const double *sT, const double *sU, const double *sA, double *sImg,
                                        int J0, int j3, int i3, int i2, int j2)
{
    using C = LoCfg<S, P>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int L = C::L, L2Q = C::L2Q, LP = C::LP, N = C::N;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n3a = C::n(A, 2);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha1 = sh_of(S, A, 1), shb1 = sh_of(S, B, 1);
    constexpr int offA = C::off(A), offB = C::off(B);
    const double *U = sU + C::uoff(A, B);
    const double *Ab = sA + C::aoff(A, B);
    // J0: first packed row of the pass's image
    {
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
        constexpr int J1U = HXG_LO_J1U;
#pragma unroll J1U
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
}

// One pass: the slabs j3lo .. j3lo + nj - 1 of trial block B (a contiguous range of packed rows)
template <int S, int P, int B>
__device__ __forceinline__ void lo_pass(const double *sT, const double *sU, const double *sM, double *sA0,
                                        double *sImg0, double *__restrict__ outE, int j3lo, int nj, int slot,
                                        int tin, bool live, int nlive)
{
    using C = LoCfg<S, P>;
    // slot-0 pointers sA0 / sImg0: stage A and the write-out work on this thread's own
    // slot, the items of stage BC on any live slot
    double *sA = sA0 + slot * C::SLOT, *sImg = sImg0 + slot * C::SLOT;
    constexpr int N = C::N;
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1), n3b = C::n(B, 2), offB = C::off(B);
    constexpr int R = n1b * n2b;
    const int J0 = offB + R * j3lo;
    if (live) {
        for (int sj = 0; sj < nj; ++sj) {
            lo_stage_a<S, P, B, B>(sT, sM, sA + sj * C::A_TOT1, j3lo + sj, tin);
            if constexpr (C::NB > 1 && B <= 1)
                lo_stage_a<S, P, B + 1 < 3 ? B + 1 : 2, B>(sT, sM, sA + sj * C::A_TOT1, j3lo + sj, tin);
            if constexpr (C::NB > 1 && B == 0) lo_stage_a<S, P, 2, B>(sT, sM, sA + sj * C::A_TOT1, j3lo + sj, tin);
        }
    }
    __syncthreads();  // Abar ready; the previous pass's image has been written out
    {
        // items of the pass, without those wholly below the diagonal, dealt to the whole CTA
        // across its element slots; per slab: diagonal pair (i3 = j3: i2 >= j2; i3 > j3: all),
        // then the pairs a > b
        constexpr int n2sq = n2b * n2b, ntri = n2b * (n2b + 1) / 2;
        constexpr int A1 = B + 1 < 3 ? B + 1 : 2;
        constexpr int NIT1 = (C::NB > 1 && B <= 1) ? C::n(A1, 2) * C::n(A1, 1) * n2b : 0;
        constexpr int NIT2 = (C::NB > 1 && B == 0) ? C::n(2, 2) * C::n(2, 1) * n2b : 0;
        // slab j3 holds tot(j3) = ntri + (n3b - 1 - j3) n2sq + NIT1 + NIT2 items
        int total = 0;
        for (int sj = 0; sj < nj; ++sj) total += ntri + (n3b - 1 - (j3lo + sj)) * n2sq + NIT1 + NIT2;
        for (int q = threadIdx.x; q < C::EB * total; q += LO_THREADS) {
            const int sl = q / total;
            int it = q - sl * total;
            if (sl >= nlive) break;
            int sj = 0, j3 = j3lo;
            for (;;) {
                const int t = ntri + (n3b - 1 - j3) * n2sq + NIT1 + NIT2;
                if (it < t) break;
                it -= t;
                ++sj;
                ++j3;
            }
            const double *sAq = sA0 + sl * C::SLOT + sj * C::A_TOT1;
            double *sImgq = sImg0 + sl * C::SLOT;
            const int nd = ntri + (n3b - 1 - j3) * n2sq;
            if (it < nd) {
                int i3, i2, j2;
                if (it < ntri) {
                    i3 = j3;
                    j2 = 0;
                    while (it >= n2b - j2) { it -= n2b - j2; ++j2; }
                    i2 = j2 + it;
                } else {
                    it -= ntri;
                    i3 = j3 + 1 + it / n2sq;
                    it -= (i3 - j3 - 1) * n2sq;
                    j2 = it / n2b;
                    i2 = it - j2 * n2b;
                }
                lo_item<S, P, B, B>(sT, sU, sAq, sImgq, J0, j3, i3, i2, j2);
            } else if (it < nd + NIT1) {
                if constexpr (NIT1 > 0) {
                    it -= nd;
                    constexpr int n2a = C::n(A1, 1);
                    const int i2 = it % n2a, r = it / n2a, j2 = r % n2b, i3 = r / n2b;
                    lo_item<S, P, A1, B>(sT, sU, sAq, sImgq, J0, j3, i3, i2, j2);
                }
            } else {
                if constexpr (NIT2 > 0) {
                    it -= nd + NIT1;
                    constexpr int n2a = C::n(2, 1);
                    const int i2 = it % n2a, r = it / n2a, j2 = r % n2b, i3 = r / n2b;
                    lo_item<S, P, 2, B>(sT, sU, sAq, sImgq, J0, j3, i3, i2, j2);
                }
            }
        }
    }
    __syncthreads();  // image complete
    if (live) {
        const int Rp = R * nj;
        const int len = Rp * N - (Rp * J0 + Rp * (Rp - 1) / 2);
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
    double *sA0 = smem + C::COMMON + ((C::NF * L3 + 1) & ~1);  // slot 0: Abar, then the slab image
    double *sImg0 = sA0 + C::A_TOT;
    for (long long e0 = (long long)blockIdx.x * C::EB; e0 < args.E; e0 += (long long)gridDim.x * C::EB) {
        const long long e = e0 + slot;
        const bool live = slot < C::EB && e < args.E;  // (threads beyond EB * TPE only deal items)
        const int nlive = (int)(args.E - e0 < C::EB ? args.E - e0 : C::EB);  // live slots of this pass
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
        for (int j3 = 0; j3 < C::n(0, 2); j3 += C::NJ3)
            lo_pass<S, P, 0>(sT, sU, sM, sA0, sImg0, outE, j3, cmin(C::NJ3, C::n(0, 2) - j3), slot, tin, live, nlive);
        if constexpr (NB > 1) {
            for (int j3 = 0; j3 < C::n(1, 2); j3 += C::NJ3)
                lo_pass<S, P, 1>(sT, sU, sM, sA0, sImg0, outE, j3, cmin(C::NJ3, C::n(1, 2) - j3), slot, tin, live, nlive);
            for (int j3 = 0; j3 < C::n(2, 2); j3 += C::NJ3)
                lo_pass<S, P, 2>(sT, sU, sM, sA0, sImg0, outE, j3, cmin(C::NJ3, C::n(2, 2) - j3), slot, tin, live, nlive);
        }
    }
}

}  // namespace hxg
