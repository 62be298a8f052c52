// hxg_general_v4.cuh -- warp-per-work-unit general-map Gram kernel for high
// orders (digit extents and L up to 16): the v3 dataflow (hxg_general_v3.cuh)
// with every 8x8 DMMA operand split into tiles.
//
//   stage A (xi3, DFMA)  Abar_g[m][l], l, m < L                      (warp smem)
//   per trial digit j2:
//     stage B (xi2, DMMA) B_h[i2][l]: tiles (i2 / 8, l / 8), K = m
//     per test-digit chunk i2 in [8c, 8c + 8):
//       stage C (xi1, DMMA) Y-form tiles (j1 / 8, i1 / 8) per i2, or
//                           B-form tiles (j1 / 8, i2 chunk) per i1
//       write-out           one cp.async.bulk per packed row segment
//                           (columns of the chunk), double-buffered staging
// Many independent accumulator chains per warp (up to 2 x 2 x 2) keep the FP64
// tensor pipe busy at the low occupancy the larger shared-memory footprint
// allows.
#pragma once
#include "hxg_common.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_general_v3.cuh"
#include "hxg_terms.h"

namespace hxg {

template <int S, int P, int L>
struct V4Cfg {
    using C2 = V2Cfg<S, P, L>;
    static constexpr int NB = C2::NB, NF = C2::NF, L3 = C2::L3, N = C2::N;
    static constexpr int NG = C2::NG, NH = C2::NH;
    __host__ __device__ static constexpr int n(int a, int d) { return C2::n(a, d); }
    static constexpr int N1 = C2::N1, N2 = C2::N2;
    static constexpr bool OK = L <= 16 && N1 <= 16 && N2 <= 16;
    static constexpr int T2 = (N2 + 7) / 8;   // i2 tiles (stage B rows)
    static constexpr int TL = (L + 7) / 8;    // l tiles (stage B columns)
    static constexpr int LQ = (L + 3) / 4;    // m k-steps
    static constexpr int SLA = 8 * TL;        // Abar / B_h row stride (l)
    static constexpr int RA = 4 * LQ;         // Abar rows (m, zero padded)
    static constexpr int NT = V3Cfg<S, P, L>::NT;
    static constexpr int LP = (L + 1) & ~1;
    static constexpr int SW = 8 * N1 + 2;     // staging row stride: an 8-digit i2 chunk
#ifndef HXG_V4_WARPS
#define HXG_V4_WARPS 4
#endif
#ifndef HXG_V4_NBUF
#define HXG_V4_NBUF 1
#endif
    static constexpr int WARPS = HXG_V4_WARPS;
    static constexpr int NBUF = HXG_V4_NBUF;  // staging buffers per warp
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int W_P = 0;                          // [NT][16]
    static constexpr int W_A = W_P + NT * 16;              // [NG][RA][SLA]
    static constexpr int W_B = W_A + NG * RA * SLA;        // [NH][8 T2][SLA]
    static constexpr int W_S = W_B + NH * 8 * T2 * SLA;    // [2][N1][SW]
    static constexpr int W_TOT = ((W_S + NBUF * N1 * SW + 1) / 2) * 2;
    static constexpr int OFF_T = 0;
    static constexpr int OFF_W = 2 * KT * LP;
    static constexpr int SMEM_BYTES = (OFF_W + WARPS * W_TOT) * 8 + 16;
    // one (j3, i3) digit pair per work unit (v3 may group several i3 per unit)
    __host__ __device__ static constexpr int pair_units(int a, int b)
    {
        return a == b ? n(a, 2) * (n(a, 2) + 1) / 2 : n(a, 2) * n(b, 2);
    }
    __host__ __device__ static constexpr int units()
    {
        int u = 0;
        for (int b = 0; b < NB; ++b)
            for (int a = b; a < NB; ++a) u += pair_units(a, b);
        return u;
    }
    static constexpr int NU = units();
    static constexpr int MINB = cmin(4, (228 * 1024) / (SMEM_BYTES + 1024));
    // stage-C factorization per block pair, FP64-pipe cost with tiles (x8):
    // B-form per 8 test digits i2: n1a x MB x NKS DMMA (+ a DMUL per lane);
    // Y-form per i2: MB x MA x KSY DMMA + MB x KSY x YQ Y-build FMAs per lane
    __host__ __device__ static constexpr bool yform(int a, int b)
    {
        const CPair pp = make_pair_plan(S, a, b);
        const int ma = (n(a, 0) + 7) / 8, mb = (n(b, 0) + 7) / 8;
        const int costB8 = n(a, 0) * mb * ((pp.nh * L + 3) / 4) * 288;
        const int ksy = (pp.nr * L + 3) / 4;
        const int costY8 = 8 * (mb * ma * ksy * 256 + mb * ksy * 32 * V2Cfg<S, P, L>::yq(a, b));
        return costY8 < costB8;
    }
};

template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void v4_unit(const V3Args &args, const double *sT, double *W,
                                        const double *__restrict__ M, double *__restrict__ outE,
                                        int epar, int j3, int i3, int &buf, unsigned &keep)
{
    using C = V4Cfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr GList GL = make_glist(pp);
    constexpr int LP = C::LP, L3 = C::L3, N = C::N, SW = C::SW, SLA = C::SLA, RA = C::RA;
    constexpr int LQ = C::LQ, TL = C::TL;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int MA = (n1a + 7) / 8, MB = (n1b + 7) / 8, T2A = (n2a + 7) / 8;
    constexpr int sha0 = sh_of(S, A, 0), sha1 = sh_of(S, A, 1), sha2 = sh_of(S, A, 2);
    constexpr int shb0 = sh_of(S, B, 0), shb1 = sh_of(S, B, 1), shb2 = sh_of(S, B, 2);
    constexpr int offA = V2Cfg<S, P, L>::off(A), offB = V2Cfg<S, P, L>::off(B);
    constexpr bool YF = C::yform(A, B);
    constexpr int ncols = n1a * n2a;
    const int lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
    double *sP = W + C::W_P, *sA = W + C::W_A, *sBw = W + C::W_B;

    // ---------------- stage A: contract xi3 ----------------
    for (int o = lane; o < pp.nt * 16; o += 32) {
        const int t = o >> 4, n = o & 15;
        int fr = 0, fs = 0;
#pragma unroll
        for (int tt = 0; tt < pp.nt; ++tt)
            if (tt == t) { fr = pp.t_fr[tt]; fs = pp.t_fs[tt]; }
        sP[o] = n < L ? sT[(fr * KT + i3 + sha2) * LP + n] * sT[(fs * KT + j3 + shb2) * LP + n] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int g = 0; g < pp.ng; ++g) {
#pragma unroll 1
        for (int lm0 = 0; lm0 < L * L; lm0 += 32) {
            const int lm = cmin(lm0 + lane, L * L - 1);
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < pp.nt; ++t) {
                if (pp.t_g[t] != g) continue;
                const double *Mf = M + pp.t_field[t] * L3 + lm;
                const double *pt = sP + t * 16;
                double v[L];
#pragma unroll
                for (int n = 0; n < L; ++n) v[n] = __ldg(Mf + n * L * L);
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int n = 0; n < L; n += 2) {
                    s0 = fma(v[n], pt[n], s0);
                    if (n + 1 < L) s1 = fma(v[n + 1], pt[n + 1], s1);
                }
                acc += pp.t_sign[t] > 0 ? (s0 + s1) : -(s0 + s1);
            }
            if (lm0 + lane < L * L) {
                const int l = lm / L, m = lm - l * L;
                sA[(g * RA + m) * SLA + l] = acc;
            }
        }
    }
    __syncwarp();

    // ---------------- per-unit operand registers ----------------
    double Ta[2][T2A][LQ];  // stage B A operand: u_fr(i2 = 8 it + g8, m = 4 ks + t4)
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
        for (int it = 0; it < T2A; ++it)
#pragma unroll
            for (int ks = 0; ks < LQ; ++ks) {
                const int m = ks * 4 + t4, i2 = it * 8 + g8;
                Ta[fr][it][ks] = (m < L && i2 < n2a) ? sT[(fr * KT + i2 + sha1) * LP + m] : 0.0;
            }
    constexpr int KD = pp.nh * L, NKS = (KD + 3) / 4;
    constexpr int YQ = V2Cfg<S, P, L>::yq(A, B);
    constexpr int KSY = (pp.nr * L + 3) / 4;
    constexpr int NK = YF ? KSY : NKS;
    double Rt[YF ? MA : MB][NK];                 // Y: u_r(i1, l)  (B operand, per i1 tile)
                                                 // B: u_s(j1, l)  (A operand, per j1 tile)
    double Yc[YF ? MB : 1][YF ? KSY : 1][YQ];    // Y: trial coefficients per j1 tile
    int Ro[NK][YF ? YQ : 1];                     // sBw offsets (h, l) [Y] / (h, l) [B]
    int Xo[YF ? 1 : NKS];                        // B: sT offset of u_r(sha0, l)
    (void)Yc;
    (void)Xo;
    if constexpr (YF) {
#pragma unroll
        for (int ks = 0; ks < KSY; ++ks) {
            const int k = ks * 4 + t4;
            const bool kv = k < pp.nr * L;
            const int r = kv ? k / L : 0, l = kv ? k - r * L : 0;
            int rc = 0;
#pragma unroll
            for (int rr = 0; rr < pp.nr; ++rr)
                if (rr == r) rc = pp.r_code[rr];
#pragma unroll
            for (int mt = 0; mt < MA; ++mt) {
                const int i1 = mt * 8 + g8;
                Rt[mt][ks] = (kv && i1 < n1a) ? sT[(rc * KT + i1 + sha0) * LP + l] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < YQ; ++q) {
#pragma unroll
                for (int mt = 0; mt < MB; ++mt) Yc[mt][ks][q] = 0.0;
                Ro[ks][q] = l;
            }
            int q = 0;
#pragma unroll
            for (int h = 0; h < pp.nh; ++h) {
                const bool mine = kv && pp.h_r[h] == r;
#pragma unroll
                for (int qq = 0; qq < YQ; ++qq)
                    if (mine && q == qq) {
#pragma unroll
                        for (int mt = 0; mt < MB; ++mt) {
                            const int j1 = mt * 8 + g8;
                            Yc[mt][ks][qq] = j1 < n1b ? sT[(pp.h_fs[h] * KT + j1 + shb0) * LP + l] : 0.0;
                        }
                        Ro[ks][qq] = h * 8 * C::T2 * SLA + l;
                    }
                q += mine ? 1 : 0;
            }
        }
    } else {
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
            const int k = ks * 4 + t4;
            const bool kv = k < KD;
            const int h = kv ? k / L : 0, l = kv ? k - h * L : 0;
            int fs = 0, fr = 0;
#pragma unroll
            for (int hh = 0; hh < pp.nh; ++hh)
                if (hh == h) { fs = pp.h_fs[hh]; fr = pp.h_fr[hh]; }
#pragma unroll
            for (int mt = 0; mt < MB; ++mt) {
                const int j1 = mt * 8 + g8;
                Rt[mt][ks] = (kv && j1 < n1b) ? sT[(fs * KT + j1 + shb0) * LP + l] : 0.0;
            }
            Ro[ks][0] = h * 8 * C::T2 * SLA + g8 * SLA + l;  // + i2 chunk base * SLA
            Xo[ks] = kv ? (fr * KT + sha0) * LP + l : 0;
        }
    }

    const int I0 = offA + ncols * i3;
    for (int j2 = 0; j2 < n2b; ++j2) {
        // ---------------- stage B: contract xi2 on DMMA ----------------
        double Tb[2][LQ];
#pragma unroll
        for (int fs = 0; fs < 2; ++fs)
#pragma unroll
            for (int ks = 0; ks < LQ; ++ks) {
                const int m = ks * 4 + t4;
                Tb[fs][ks] = m < L ? sT[(fs * KT + j2 + shb1) * LP + m] : 0.0;
            }
#pragma unroll
        for (int h = 0; h < pp.nh; ++h) {
            double d[T2A][TL][2];
#pragma unroll
            for (int it = 0; it < T2A; ++it)
#pragma unroll
                for (int lt = 0; lt < TL; ++lt) d[it][lt][0] = d[it][lt][1] = 0.0;
#pragma unroll
            for (int q = 0; q < MAXG; ++q) {
                const int g = GL.g[h][q];
                if (g < 0) continue;
#pragma unroll
                for (int ks = 0; ks < LQ; ++ks) {
                    double bv[TL];
#pragma unroll
                    for (int lt = 0; lt < TL; ++lt) bv[lt] = sA[(g * RA + ks * 4 + t4) * SLA + lt * 8 + g8];
#pragma unroll
                    for (int it = 0; it < T2A; ++it) {
                        const double av = Ta[pp.g_fr[g]][it][ks] * Tb[pp.g_fs[g]][ks];
#pragma unroll
                        for (int lt = 0; lt < TL; ++lt)
                            dmma_8x8x4_keep(d[it][lt][0], d[it][lt][1], av, bv[lt], keep);
                    }
                }
            }
#pragma unroll
            for (int it = 0; it < T2A; ++it)
#pragma unroll
                for (int lt = 0; lt < TL; ++lt) {
                    double *dst = sBw + (h * 8 * C::T2 + it * 8 + g8) * SLA + lt * 8 + 2 * t4;
                    dst[0] = d[it][lt][0];
                    dst[1] = d[it][lt][1];
                }
        }
        __syncwarp();
#pragma unroll 1
        for (int c0 = 0; c0 < n2a; c0 += 8) {  // test-digit chunk i2 in [c0, c0 + 8)
            const int cn = cmin(8, n2a - c0);
            const int ccols = cn * n1a;
            if constexpr (C::NBUF == 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
            double *sS = W + C::W_S + (C::NBUF == 2 ? buf : 0) * C::N1 * SW;
            const int Ic = I0 + c0 * n1a;  // first column of the chunk
            // ---------------- stage C: contract xi1 on DMMA ----------------
            if constexpr (YF) {
#pragma unroll 1
                for (int i2 = c0; i2 < c0 + cn; i2 += 2) {
                    const bool two = i2 + 1 < c0 + cn;
                    double d[2][MB][MA][2];
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int mt = 0; mt < MB; ++mt)
#pragma unroll
                            for (int nt = 0; nt < MA; ++nt) d[c][mt][nt][0] = d[c][mt][nt][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < KSY; ++ks) {
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            if (c == 1 && !two) continue;
                            const double *base = sBw + (i2 + c) * SLA;
                            double bq[YQ];
#pragma unroll
                            for (int q = 0; q < YQ; ++q) bq[q] = base[Ro[ks][q]];
#pragma unroll
                            for (int mt = 0; mt < MB; ++mt) {
                                double y = Yc[mt][ks][0] * bq[0];
#pragma unroll
                                for (int q = 1; q < YQ; ++q) y = fma(Yc[mt][ks][q], bq[q], y);
#pragma unroll
                                for (int nt = 0; nt < MA; ++nt)
                                    dmma_8x8x4_keep(d[c][mt][nt][0], d[c][mt][nt][1], y, Rt[nt][ks], keep);
                            }
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c == 1 && !two) continue;
#pragma unroll
                        for (int mt = 0; mt < MB; ++mt) {
                            const int j1 = mt * 8 + g8;
                            if (j1 >= n1b) continue;
                            const int J = offB + j1 + n1b * (j2 + n2b * j3);
                            const int pad = (epar + J * N - J * (J - 1) / 2 - J + Ic) & 1;
                            double *srow = sS + j1 * SW + pad + (i2 + c - c0) * n1a;
#pragma unroll
                            for (int nt = 0; nt < MA; ++nt) {
                                const int i1 = nt * 8 + 2 * t4;
                                if (i1 < n1a) srow[i1] = d[c][mt][nt][0];
                                if (i1 + 1 < n1a) srow[i1 + 1] = d[c][mt][nt][1];
                            }
                        }
                    }
                }
            } else {
#pragma unroll 1
                for (int i1 = 0; i1 < n1a; ++i1) {
                    double d[MB][2];
#pragma unroll
                    for (int mt = 0; mt < MB; ++mt) d[mt][0] = d[mt][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < NKS; ++ks) {
                        const double bv = sT[Xo[ks] + i1 * LP] * sBw[Ro[ks][0] + c0 * SLA];
#pragma unroll
                        for (int mt = 0; mt < MB; ++mt) dmma_8x8x4_keep(d[mt][0], d[mt][1], Rt[mt][ks], bv, keep);
                    }
#pragma unroll
                    for (int mt = 0; mt < MB; ++mt) {
                        const int j1 = mt * 8 + g8;
                        if (j1 >= n1b) continue;
                        const int J = offB + j1 + n1b * (j2 + n2b * j3);
                        const int pad = (epar + J * N - J * (J - 1) / 2 - J + Ic) & 1;
                        double *srow = sS + j1 * SW + pad;
                        if (2 * t4 < cn) srow[(2 * t4) * n1a + i1] = d[mt][0];
                        if (2 * t4 + 1 < cn) srow[(2 * t4 + 1) * n1a + i1] = d[mt][1];
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            // ---------------- write-out: lane j1 copies its row's chunk ----------------
            if (lane < n1b) {
                const int j1 = lane;
                const int J = offB + j1 + n1b * (j2 + n2b * j3);
                const int goff = J * N - J * (J - 1) / 2 - J + Ic;
                const int pad = (epar + goff) & 1;
                const int cs = J > Ic ? J - Ic : 0;
                if (cs < ccols) {
                    const double *src = sS + j1 * SW + pad + cs;
                    double *dst = outE + goff + cs;
                    int len = ccols - cs;
                    if (reinterpret_cast<size_t>(dst) & 8) {
                        __stcs(dst, *src);
                        ++dst;
                        ++src;
                        --len;
                    }
                    if (len & 1) __stcs(dst + len - 1, src[len - 1]);
                    if (len >= 2) bulk_s2g(dst, src, (len & ~1) * 8);
                }
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            buf ^= 1;
            __syncwarp();
        }
    }
}

template <int S, int P, int L>
__global__ void __launch_bounds__(V4Cfg<S, P, L>::THREADS, (V4Cfg<S, P, L>::MINB))
    general_v4_kernel(const __grid_constant__ V3Args args)
{
    using C = V4Cfg<S, P, L>;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_next;
    const int e = blockIdx.x / args.split;
    const int part = blockIdx.x - e * args.split;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sT = smem + C::OFF_T;
    for (int idx = threadIdx.x; idx < 2 * KT * C::LP; idx += C::THREADS) {
        const int fk = idx / C::LP, l = idx - fk * C::LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    double *W = smem + C::OFF_W + warp * C::W_TOT;
    for (int idx = lane; idx < C::W_TOT; idx += 32) W[idx] = 0.0;
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    const double *__restrict__ M = args.metric + (long long)e * C::NF * C::L3;
    double *__restrict__ outE = args.out + (long long)e * args.P;
    const int epar = (int)((reinterpret_cast<size_t>(outE) >> 3) & 1);
    const int lo = (int)((long long)C::NU * part / args.split);
    const int hi = (int)((long long)C::NU * (part + 1) / args.split);
    int buf = 0;
    unsigned keep = 0;
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&s_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0) + lo;
        if (u >= hi) break;
        int rem = u, pair = -1, j3 = 0, i3 = 0;
#pragma unroll
        for (int b = 0; b < C::NB; ++b)
#pragma unroll
            for (int a = b; a < C::NB; ++a) {
                if (pair < 0) {
                    const int cnt = C::pair_units(a, b);
                    if (rem < cnt) {
                        pair = a * 3 + b;
                        if (a == b) {
                            const int n3 = C::n(a, 2);
                            int jj = 0, r = rem;
                            while (r >= n3 - jj) { r -= n3 - jj; ++jj; }
                            j3 = jj;
                            i3 = jj + r;
                        } else {
                            j3 = rem / C::n(a, 2);
                            i3 = rem - j3 * C::n(a, 2);
                        }
                    } else {
                        rem -= cnt;
                    }
                }
            }
        if constexpr (C::NB == 1) {
            v4_unit<S, P, L, 0, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep);
        } else {
            switch (pair) {
            case 0: v4_unit<S, P, L, 0, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            case 3: v4_unit<S, P, L, 1, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            case 6: v4_unit<S, P, L, 2, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            case 4: v4_unit<S, P, L, 1, 1>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            case 7: v4_unit<S, P, L, 2, 1>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            default: v4_unit<S, P, L, 2, 2>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
            }
        }
    }
    if (args.E < 0 && keep == 0x9e3779b9u) args.out[0] = keep;
    bulk_wait_all();
}

}  // namespace hxg
