// hxg_general_v3.cuh -- warp-per-work-unit general-map Gram kernel
// (compile-time space / order / rule; orders with every digit extent <= 8 and
// L <= 8, i.e. the BASELINE configs 1-4).
//
// Each warp owns one work unit at a time -- (element e, trial block b, test
// block a >= b, digits j3, i3) -- and runs all three sum-factorization stages
// for it with warp-private shared memory, so no CTA-wide barrier ever stalls
// the FP64 pipe:
//   stage A (xi3, DFMA)   Abar_g[m][l] = sum_t sign_t sum_n M_t[n][l,m] u(i3,n) u(j3,n)
//   for every trial digit j2:
//     stage B (xi2, DMMA) B_h[i2][l] = sum_{g in h} sum_m V_g[i2][m] Abar_g[m][l]
//     stage C (xi1, DMMA) Y-form or B-form (see hxg_general_v2.cuh), one 8x8
//                         tile per test digit i2 (Y) or i1 (B)
//     write-out           one bulk copy (cp.async.bulk, TMA engine) per packed
//                         row segment, double-buffered staging
// CTAs of 4 warps take the work units of one element from a shared-memory
// counter (dynamic balancing; the element's metric stays L1/L2-resident).
#pragma once
#include "hxg_common.cuh"
#include "hxg_geom.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_terms.h"

namespace hxg {

#ifndef HXG_V3_DEBUG_EMIN
#define HXG_V3_DEBUG_EMIN 0
#endif
#ifndef HXG_V3_AFRAG
#define HXG_V3_AFRAG 1  // Abar in stage-B fragment order (0: row-major [m][l], 2-way bank conflicts)
#endif
#ifndef HXG_V3_TF
#define HXG_V3_TF 4
#endif
constexpr int kTF = HXG_V3_TF;  // stage-C output tiles in flight per warp
#if defined(HXG_V3_DEBUG) || defined(HXG_V3_DEBUG2)
__device__ double *hxg_dbg;
#endif
constexpr int V3_WARPS = 4;
constexpr int V3_THREADS = V3_WARPS * 32;

template <int S, int P, int L>
struct V3Cfg {
    using C2 = V2Cfg<S, P, L>;
    static constexpr int NB = C2::NB, NF = C2::NF, L3 = C2::L3, N = C2::N;
    static constexpr int NG = C2::NG, NH = C2::NH, C12 = C2::C12;
    __host__ __device__ static constexpr int n(int a, int d) { return C2::n(a, d); }
    static constexpr bool OK = L <= 8 && C2::N1 <= 8 && C2::N2 <= 8;
    __host__ __device__ static constexpr int maxt()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b < NB; ++b) m = cmax(m, make_pair_plan(S, a, b).nt);
        return m;
    }
    static constexpr int NT = maxt();
    // test digits i3 per work unit: the packed row segment of a unit is K * C12 long, so
    // each bulk copy moves K times as many bytes and the issuing warp spends K times
    // fewer copy-issue cycles (the UBLKCP waterfall) per output byte (DESIGN.md,
    // "Write-out cost"); HBM-bound spaces use K > 1 with one staging buffer,
    // FP64-bound spaces K = 1 with two
    // measured best of K = 1..4 (profiles/v3_k_r01.txt, sweep_r01.json): H(div) 4 at
    // p <= 4 and p = 7, 2 at p = 6, 1 at p = 5; L2 (p = 7) 4
#ifdef HXG_V3_K_HDIV
    static constexpr int KHD = HXG_V3_K_HDIV;
#else
    static constexpr int KHD = P == 5 ? 1 : (P == 6 ? 2 : 4);
#endif
#ifndef HXG_V3_K_L2
#define HXG_V3_K_L2 4
#endif
    static constexpr int K = P <= 2 ? 1 : (S == HDIV ? KHD : (S == L2 ? HXG_V3_K_L2 : 1));
    static constexpr int NSTG = K == 1 ? 2 : 1;  // staging buffers per warp
    static constexpr int LP = (L + 1) & ~1;      // sT row stride
    static constexpr int SW = ((K * C12 + 1 + 1) / 2) * 2;  // staging row stride (even, >= K C12 + 1)
    // per-warp shared memory (doubles)
    static constexpr int W_P = 0;                       // [NT][8]   stage-A 1D products
    static constexpr int W_A = W_P + NT * 8;            // [K][NG][8][8] Abar (rows m, cols l; zero padded)
    static constexpr int W_B = W_A + K * NG * 64;       // [NH][8][8] B_h (rows i2, cols l)
    static constexpr int W_S = W_B + NH * 64;           // [NSTG][N1][SW] staging
    static constexpr int W_TOT = W_S + NSTG * C2::N1 * SW;
    static constexpr int OFF_T = 0;                     // CTA-shared [2][KT][LP]
    static constexpr int OFF_W = 2 * KT * LP;
    // p <= 3: the element's metric fields are evaluated in the kernel into shared
    // memory (the separate metric pass would move as many bytes as the output)
    static constexpr bool FUSED = P <= 3;
    static constexpr int OFF_M = OFF_W + V3_WARPS * W_TOT;
    static constexpr int SMEM_BYTES = (OFF_M + (FUSED ? NF * L3 : 0)) * 8 + 16;
    __host__ __device__ static constexpr int kcnt(int r) { return (r + K - 1) / K; }  // units over r digits i3
    __host__ __device__ static constexpr int pair_units(int a, int b)
    {
        int u = 0;
        for (int j3 = 0; j3 < n(b, 2); ++j3) u += kcnt(a == b ? n(a, 2) - j3 : n(a, 2));
        return u;
    }
    __host__ __device__ static constexpr int units()
    {
        int u = 0;
        for (int b = 0; b < NB; ++b)
            for (int a = b; a < NB; ++a) u += pair_units(a, b);
        return u;
    }
    static constexpr int NU = units();
#ifdef HXG_V3_MINB
    static constexpr int MINB = HXG_V3_MINB;
#else
    // CTAs per SM: 5 (<= 102 registers) measured best for H1/H(curl), 4 for H(div) and L2
    static constexpr int MINB = cmin((S == L2 || S == HDIV) ? 4 : 5, (228 * 1024) / (SMEM_BYTES + 1024));
#endif
};

struct V3Args {
    const double *tables;
    const double *metric;  // [E][nfields][n][l][m]; NULL for the fused low-order path
    double *out;
    long long P;
    int E;
    int split;  // CTAs per element
    int range;  // 1: CTA c owns the contiguous (element, unit) items [c T / G, (c + 1) T / G), T = E * NU
    // fused low-order path (C::FUSED): geometry evaluated in the kernel
    const int *kind;
    const double *params, *coef, *wgrid;
    int *status;
};

// metric field load: shared memory on the fused path, read-only global otherwise
template <bool FUSED>
__device__ __forceinline__ double metric_ld(const double *p)
{
    if constexpr (FUSED) return *p;
    else return __ldg(p);
}

// stage-B groups listed per h: gl[h][q] = q-th g with g_h[g] == h, or -1
struct GList {
    int g[MAXH][MAXG];
};
__host__ __device__ constexpr GList make_glist(const CPair &pp)
{
    GList L{};
    for (int h = 0; h < MAXH; ++h) {
        int q = 0;
        for (int k = 0; k < MAXG; ++k) L.g[h][k] = -1;
        for (int g = 0; g < pp.ng; ++g)
            if (pp.g_h[g] == h) L.g[h][q++] = g;
    }
    return L;
}

// explicit shared-memory load (ordered after the warp barrier that publishes B_h)
__device__ __forceinline__ double lds_f64(const double *p)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}

template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void v3_unit(const V3Args &args, const double *sT, double *W,
                                        const double *__restrict__ M, double *__restrict__ outE,
                                        int epar, int j3, int i3, int &buf, unsigned &keep)
{
    using C = V3Cfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr GList GL = make_glist(pp);
    constexpr int LP = C::LP, L3 = C::L3, N = C::N, SW = C::SW;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha0 = sh_of(S, A, 0), sha1 = sh_of(S, A, 1), sha2 = sh_of(S, A, 2);
    constexpr int shb0 = sh_of(S, B, 0), shb1 = sh_of(S, B, 1), shb2 = sh_of(S, B, 2);
    constexpr int offA = V2Cfg<S, P, L>::off(A), offB = V2Cfg<S, P, L>::off(B);
    constexpr bool YF = V2Cfg<S, P, L>::yform(A, B);
    constexpr int LQ = (L + 3) / 4;  // k-steps over a length-L contraction
    constexpr int ncols = n1a * n2a;
    const int lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
    double *sP = W + C::W_P, *sA = W + C::W_A, *sBw = W + C::W_B;

    constexpr int K = C::K;
    constexpr int n3a = C::n(A, 2);
    const int kc = cmin(K, n3a - i3);  // test digits i3 .. i3 + kc - 1 in this unit
    // ---------------- stage A: contract xi3 (per test digit of the unit) ----------------
    for (int kk = 0; kk < K; ++kk) {
    if (kk >= kc) break;
    const int i3k = i3 + kk;
    double *sAk = sA + kk * C::NG * 64;
    __syncwarp();
    for (int o = lane; o < pp.nt * 8; o += 32) {
        const int t = o >> 3, n = o & 7;
        int fr = 0, fs = 0;
#pragma unroll
        for (int tt = 0; tt < pp.nt; ++tt)
            if (tt == t) { fr = pp.t_fr[tt]; fs = pp.t_fs[tt]; }
        sP[o] = n < L ? sT[(fr * KT + i3k + sha2) * LP + n] * sT[(fs * KT + j3 + shb2) * LP + n] : 0.0;
    }
    __syncwarp();
    constexpr int NPASS = (L * L + 31) / 32;  // metric points per lane
#pragma unroll
    for (int g = 0; g < pp.ng; ++g) {
        double acc[NPASS];
#pragma unroll
        for (int q = 0; q < NPASS; ++q) acc[q] = 0.0;
#pragma unroll
        for (int t = 0; t < pp.nt; ++t) {
            if (pp.t_g[t] != g) continue;
            const double *Mf = M + pp.t_field[t] * L3;
            const double *pt = sP + t * 8;
            double v[NPASS][L];
#pragma unroll
            for (int q = 0; q < NPASS; ++q) {
                const int lm = cmin(lane + 32 * q, L * L - 1);
#pragma unroll
                for (int n = 0; n < L; ++n) v[q][n] = metric_ld<C::FUSED>(Mf + n * L * L + lm);
            }
#pragma unroll
            for (int q = 0; q < NPASS; ++q) {
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int n = 0; n < L; n += 2) {
                    s0 = fma(v[q][n], pt[n], s0);
                    if (n + 1 < L) s1 = fma(v[q][n + 1], pt[n + 1], s1);
                }
                acc[q] += pp.t_sign[t] > 0 ? (s0 + s1) : -(s0 + s1);
            }
        }
#pragma unroll
        for (int q = 0; q < NPASS; ++q) {
            const int lm = lane + 32 * q;
            if (lm < L * L) {
                const int l = lm / L, m = lm - l * L;
                // stage-B B fragment order (k = m, n = l): conflict-free 8-byte loads
                if constexpr (HXG_V3_AFRAG) sAk[g * 64 + (m >> 2) * 32 + l * 4 + (m & 3)] = acc[q];
                else sAk[(g * 8 + m) * 8 + l] = acc[q];
            }
        }
    }
    }  // kk
    __syncwarp();

    // ---------------- per-unit operand registers ----------------
    // stage B: A operand V_g[i2 = g8][m] = u_{fr}(i2, m) * u_{fs}(j2, m); Ta = test factor
    double Ta[2][LQ];
#pragma unroll
    for (int fr = 0; fr < 2; ++fr)
#pragma unroll
        for (int ks = 0; ks < LQ; ++ks) {
            const int m = ks * 4 + t4;
            Ta[fr][ks] = (m < L && g8 < n2a) ? sT[(fr * KT + g8 + sha1) * LP + m] : 0.0;
        }
    // stage C operands
    constexpr int KD = pp.nh * L, NKS = (KD + 3) / 4;
    constexpr int YQ = V2Cfg<S, P, L>::yq(A, B);
    constexpr int KSY = (pp.nr * L + 3) / 4;
    constexpr int NR1 = YF ? KSY : NKS;
    double R0[NR1];   // Y: Yb (u_r(i1 = g8, l))   B: Af (u_s(j1 = g8, l))
    double Yc[YF ? KSY : 1][YQ];
    int Ro[NR1][YF ? YQ : 1];  // Y: sBw offsets per factor   B: sBw offset (h, i2 = g8, l)
    int Xo[YF ? 1 : NKS];      // B: sT offset of u_r(0 + sha0, l) for the test factor
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
            R0[ks] = (kv && g8 < n1a) ? sT[(rc * KT + g8 + sha0) * LP + l] : 0.0;
#pragma unroll
            for (int q = 0; q < YQ; ++q) {
                Yc[ks][q] = 0.0;
                Ro[ks][q] = l;
            }
            int q = 0;
#pragma unroll
            for (int h = 0; h < pp.nh; ++h) {
                const bool mine = kv && pp.h_r[h] == r;
#pragma unroll
                for (int qq = 0; qq < YQ; ++qq)
                    if (mine && q == qq) {
                        Yc[ks][qq] = g8 < n1b ? sT[(pp.h_fs[h] * KT + g8 + shb0) * LP + l] : 0.0;
                        Ro[ks][qq] = h * 64 + l;
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
            R0[ks] = (kv && g8 < n1b) ? sT[(fs * KT + g8 + shb0) * LP + l] : 0.0;
            Ro[ks][0] = h * 64 + g8 * 8 + l;
            Xo[ks] = kv ? (fr * KT + sha0) * LP + l : 0;  // invalid k: A operand is 0
        }
    }

    const int I0 = offA + ncols * i3;
    const int ncu = kc * ncols;  // columns of this unit's row segments
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
        const int J = offB + g8 + n1b * (j2 + n2b * j3);  // row of this lane's j1 = g8
        const int goff = J * N - J * (J - 1) / 2 - J + I0;
        const int pad = (epar + goff) & 1;
        double *sS = W + C::W_S + (C::NSTG == 2 ? buf : 0) * C::C2::N1 * SW;
        for (int kk = 0; kk < K; ++kk) {
        if (kk >= kc) break;
        const double *sAk = sA + kk * C::NG * 64;
        if (kk > 0) __syncwarp();  // previous digit's stage C has read B_h
        // two h chains at a time: independent DMMA accumulators hide the DMMA latency
#pragma unroll
        for (int h0 = 0; h0 < pp.nh; h0 += 2) {
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int q = 0; q < MAXG * LQ; ++q) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int g = (h0 + c < MAXH) ? GL.g[h0 + c][q / LQ] : -1, ks = q % LQ;
                    if (h0 + c < pp.nh && g >= 0) {
                        const double av = Ta[pp.g_fr[g]][ks] * Tb[pp.g_fs[g]][ks];
                        const double bv = HXG_V3_AFRAG ? sAk[g * 64 + ks * 32 + lane] : sAk[(g * 8 + ks * 4 + t4) * 8 + g8];
                        dmma_8x8x4_keep(d[c][0], d[c][1], av, bv, keep);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if (h0 + c < pp.nh) {
                    // one 16-byte store per lane (a row of 8 doubles per g8: 4 wavefronts, no conflicts)
                    *reinterpret_cast<double2 *>(sBw + ((h0 + c) * 8 + g8) * 8 + 2 * t4) = make_double2(d[c][0], d[c][1]);
                }
        }
        __syncwarp();
        if (kk == 0) {
            // staging buffer `buf` was last read by the bulk copies issued two row groups ago
            // (NSTG == 2) or by the previous row group's copies (NSTG == 1)
            if constexpr (C::NSTG == 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
        }
        double *srow = sS + g8 * SW + pad + kk * ncols;
        // ---------------- stage C: contract xi1 on DMMA ----------------
        if constexpr (YF) {
#pragma unroll
            for (int i2 = 0; i2 < n2a; i2 += kTF) {  // kTF tiles (i2, i2 + 1, ...) in flight
                __syncwarp();  // converged for mma.sync (.aligned) after the previous iteration's divergent stores
                double d[kTF][2];
#pragma unroll
                for (int c = 0; c < kTF; ++c) d[c][0] = d[c][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KSY; ++ks) {
#pragma unroll
                    for (int c = 0; c < kTF; ++c) {
                        if (i2 + c < n2a) {
                            const double *base = sBw + (i2 + c) * 8;
                            double y = Yc[ks][0] * base[Ro[ks][0]];
#pragma unroll
                            for (int q = 1; q < YQ; ++q) y = fma(Yc[ks][q], base[Ro[ks][q]], y);
                            dmma_8x8x4_keep(d[c][0], d[c][1], y, R0[ks], keep);
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < kTF; ++c)
                    if (i2 + c < n2a && g8 < n1b) {
                        if (2 * t4 < n1a) srow[(i2 + c) * n1a + 2 * t4] = d[c][0];
                        if (2 * t4 + 1 < n1a) srow[(i2 + c) * n1a + 2 * t4 + 1] = d[c][1];
                    }
            }
        } else {
#pragma unroll
            for (int i1 = 0; i1 < n1a; i1 += kTF) {  // kTF tiles (i1, i1 + 1, ...) in flight
                __syncwarp();  // converged for mma.sync (.aligned) after the previous iteration's divergent stores
                double d[kTF][2];
#pragma unroll
                for (int c = 0; c < kTF; ++c) d[c][0] = d[c][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < NKS; ++ks) {
                    const double bb = sBw[Ro[ks][0]];
#pragma unroll
                    for (int c = 0; c < kTF; ++c)
                        if (i1 + c < n1a)
                            dmma_8x8x4_keep(d[c][0], d[c][1], R0[ks], sT[Xo[ks] + (i1 + c) * LP] * bb, keep);
                }
#pragma unroll
                for (int c = 0; c < kTF; ++c)
                    if (i1 + c < n1a && g8 < n1b) {  // columns i2 = 2 t4, 2 t4 + 1
                        if (2 * t4 < n2a) srow[(2 * t4) * n1a + i1 + c] = d[c][0];
                        if (2 * t4 + 1 < n2a) srow[(2 * t4 + 1) * n1a + i1 + c] = d[c][1];
                    }
            }
        }
        }  // kk
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        // ---------------- write-out: lane j1 copies packed row J from column max(J, I0) ----------------
#ifdef HXG_V3_SIMPLE_WO
        for (int j1 = 0; j1 < n1b; ++j1) {
            const int Jr = offB + j1 + n1b * (j2 + n2b * j3);
            const int goffr = Jr * N - Jr * (Jr - 1) / 2 - Jr + I0;
            const int padr = (epar + goffr) & 1;
            const int csr = Jr > I0 ? Jr - I0 : 0;
            const double *srcr = sS + j1 * SW + padr;
            for (int c = csr + lane; c < ncu; c += 32) outE[goffr + c] = srcr[c];
        }
        if (false) {
#else
        if (g8 < n1b && t4 == 0) {
#endif
            const int cs = J > I0 ? J - I0 : 0;
            if (cs < ncu) {
                const double *src = sS + g8 * SW + pad + cs;
                double *dst = outE + goff + cs;
                int len = ncu - cs;
                if (reinterpret_cast<size_t>(dst) & 8) {
                    __stcs(dst, *src);
                    ++dst;
                    ++src;
                    --len;
                }
                if (len & 1) __stcs(dst + len - 1, src[len - 1]);
#ifdef HXG_V3_NO_BULK
                for (int c = 0; c < (len & ~1); ++c) __stcs(dst + c, src[c]);
#elif defined(HXG_V3_SKIP_W)  // timing experiment only: no bulk write-out
#else
                if (len >= 2) bulk_s2g(dst, src, (len & ~1) * 8);
#endif
            }
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        if constexpr (C::NSTG == 2) buf ^= 1;
        __syncwarp();  // reconverge after the divergent write-out: the next mma.sync needs the full warp
    }
#ifdef HXG_V3_DEBUG2
    if (blockIdx.x == 0 && j3 == 0 && i3 == 0 && args.E > HXG_V3_DEBUG_EMIN) {
#if HXG_V3_DEBUG2 & 1
        for (int q = lane; q < C::NG * 64; q += 32) hxg_dbg[q] = sA[q];
        for (int q = lane; q < C::NH * 64; q += 32) hxg_dbg[1024 + q] = sBw[q];
#endif
#if HXG_V3_DEBUG2 & 2
        if constexpr (YF) {
            for (int ks = 0; ks < KSY; ++ks) {
                hxg_dbg[2048 + ks * 32 + lane] = R0[ks];
                hxg_dbg[2304 + ks * 32 + lane] = Yc[ks][0];
                hxg_dbg[2560 + ks * 32 + lane] = Yc[ks][YQ - 1];
                hxg_dbg[2816 + ks * 32 + lane] = Ro[ks][0];
                hxg_dbg[3072 + ks * 32 + lane] = Ro[ks][YQ - 1];
            }
        }
#endif
#if HXG_V3_DEBUG2 & 4
        const double *sSl = W + C::W_S + (buf ^ 1) * C::C2::N1 * SW;
        for (int q = lane; q < C::C2::N1 * SW; q += 32) hxg_dbg[3328 + q] = sSl[q];
#endif
    }
#endif
}

// Low orders (p <= 2): the same unit loop with stages B and C on DFMA.  With
// digit extents <= 4 an 8x8 DMMA tile would be mostly padding, so each lane
// evaluates whole B_h values and whole Gram entries and stores the entries
// directly (consecutive lanes -> consecutive packed columns of one row).
template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void v3s_unit(const double *sT, double *W, const double *__restrict__ M,
                                         double *__restrict__ outE, int j3, int i3)
{
    using C = V3Cfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int LP = C::LP, L3 = C::L3, N = C::N;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha0 = sh_of(S, A, 0), sha1 = sh_of(S, A, 1), sha2 = sh_of(S, A, 2);
    constexpr int shb0 = sh_of(S, B, 0), shb1 = sh_of(S, B, 1), shb2 = sh_of(S, B, 2);
    constexpr int offA = V2Cfg<S, P, L>::off(A), offB = V2Cfg<S, P, L>::off(B);
    const int lane = threadIdx.x & 31;
    double *sP = W + C::W_P, *sA = W + C::W_A, *sBw = W + C::W_B;
    auto T = [&](int f, int k, int l) { return sT[(f * KT + k) * LP + l]; };

    // stage A (xi3): Abar_g[m][l]
    for (int o = lane; o < pp.nt * 8; o += 32) {
        const int t = o >> 3, n = o & 7;
        int fr = 0, fs = 0;
#pragma unroll
        for (int tt = 0; tt < pp.nt; ++tt)
            if (tt == t) { fr = pp.t_fr[tt]; fs = pp.t_fs[tt]; }
        sP[o] = n < L ? T(fr, i3 + sha2, n) * T(fs, j3 + shb2, n) : 0.0;
    }
    __syncwarp();
    if (lane < L * L) {
        const int l = lane / L, m = lane - l * L;
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < pp.nt; ++t) {
                if (pp.t_g[t] != g) continue;
                const double *Mf = M + pp.t_field[t] * L3 + lane;
                double s = 0.0;
#pragma unroll
                for (int n = 0; n < L; ++n) s = fma(metric_ld<C::FUSED>(Mf + n * L * L), sP[t * 8 + n], s);
                acc += pp.t_sign[t] > 0 ? s : -s;
            }
            sA[(g * 8 + m) * 8 + l] = acc;
        }
    }
    __syncwarp();
    const int I0 = offA + n1a * n2a * i3;
    for (int j2 = 0; j2 < n2b; ++j2) {
        // stage B (xi2): B_h[i2][l]
        for (int o = lane; o < n2a * L; o += 32) {
            const int i2 = o / L, l = o - i2 * L;
            double acc[MAXH] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int g = 0; g < pp.ng; ++g) {
                double s = 0.0;
#pragma unroll
                for (int m = 0; m < L; ++m)
                    s = fma(T(pp.g_fr[g], i2 + sha1, m) * T(pp.g_fs[g], j2 + shb1, m), sA[(g * 8 + m) * 8 + l], s);
                acc[pp.g_h[g]] += s;
            }
#pragma unroll
            for (int h = 0; h < pp.nh; ++h) sBw[(h * 8 + i2) * 8 + l] = acc[h];
        }
        __syncwarp();
        // stage C (xi1): entries of rows J = (j1, j2, j3, b), columns (i1, i2, i3, a)
        for (int o = lane; o < n1b * n2a * n1a; o += 32) {
            const int j1 = o / (n2a * n1a), r = o - j1 * (n2a * n1a);
            const int i2 = r / n1a, i1 = r - i2 * n1a;
            const int J = offB + j1 + n1b * (j2 + n2b * j3);
            const int I = I0 + r;
            if (I < J) continue;
            double v = 0.0;
#pragma unroll
            for (int h = 0; h < pp.nh; ++h)
#pragma unroll
                for (int l = 0; l < L; ++l)
                    v = fma(T(pp.h_fs[h], j1 + shb0, l) * T(pp.h_fr[h], i1 + sha0, l), sBw[(h * 8 + i2) * 8 + l], v);
            __stcs(outE + (J * N - J * (J - 1) / 2 + (I - J)), v);
        }
        __syncwarp();
    }
}

template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void v3_pick(const V3Args &args, const double *sT, double *W,
                                        const double *__restrict__ M, double *__restrict__ outE,
                                        int epar, int j3, int i3, int &buf, unsigned &keep)
{
    if constexpr (P <= 2) v3s_unit<S, P, L, A, B>(sT, W, M, outE, j3, i3);
    else v3_unit<S, P, L, A, B>(args, sT, W, M, outE, epar, j3, i3, buf, keep);
}

// decode work unit u of one element into (b, a) pair and (j3, i3), then run it
template <int S, int P, int L>
__device__ __forceinline__ void v3_run_unit(int u, const V3Args &args, const double *sT, double *W,
                                            const double *__restrict__ M, double *__restrict__ outE,
                                            int epar, int &buf, unsigned &keep)
{
    using C = V3Cfg<S, P, L>;
    // decode (b, a) pair, then (j3, i3)
    int rem = u, pair = -1, j3 = 0, i3 = 0;
#pragma unroll
    for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int a = b; a < C::NB; ++a) {
            if (pair < 0) {
                const int cnt = C::pair_units(a, b);
                if (rem < cnt) {
                    pair = a * 3 + b;
                    const int n3 = C::n(a, 2);
                    if (a == b) {  // j3 <= i3 < n3, i3 = j3 + K r
                        int jj = 0, r = rem;
                        while (r >= C::kcnt(n3 - jj)) { r -= C::kcnt(n3 - jj); ++jj; }
                        j3 = jj;
                        i3 = jj + C::K * r;
                    } else {
                        j3 = rem / C::kcnt(n3);
                        i3 = C::K * (rem - j3 * C::kcnt(n3));
                    }
                } else {
                    rem -= cnt;
                }
            }
        }
    if constexpr (C::NB == 1) {
        v3_pick<S, P, L, 0, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep);
    } else {
        switch (pair) {
        case 0: v3_pick<S, P, L, 0, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        case 3: v3_pick<S, P, L, 1, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        case 6: v3_pick<S, P, L, 2, 0>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        case 4: v3_pick<S, P, L, 1, 1>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        case 7: v3_pick<S, P, L, 2, 1>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        default: v3_pick<S, P, L, 2, 2>(args, sT, W, M, outE, epar, j3, i3, buf, keep); break;
        }
    }
}

template <int S, int P, int L>
__global__ void __launch_bounds__(V3_THREADS, (V3Cfg<S, P, L>::MINB))
    general_v3_kernel(const __grid_constant__ V3Args args)
{
    using C = V3Cfg<S, P, L>;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_next;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sT = smem + C::OFF_T;
    for (int idx = threadIdx.x; idx < 2 * KT * C::LP; idx += V3_THREADS) {
        const int fk = idx / C::LP, l = idx - fk * C::LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    double *W = smem + C::OFF_W + warp * C::W_TOT;
    for (int idx = lane; idx < C::W_TOT; idx += 32) W[idx] = 0.0;  // zero padding of Abar/B_h
    int buf = 0;
    unsigned keep = 0;  // see dmma_8x8x4_keep
#ifndef HXG_V3_FLOW
#define HXG_V3_FLOW 1
#endif
    if (HXG_V3_FLOW && !C::FUSED && args.split == 1 && args.range) {
        // one wave of CTAs, equal shares of the (element, unit) items down to one unit: no
        // tail of CTAs that drew one element more than the others (1024-element batches
        // are ~3.5 elements per resident CTA)
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        const long long T = (long long)args.E * C::NU;
        const long long lo = T * blockIdx.x / gridDim.x, hi = T * (blockIdx.x + 1) / gridDim.x;
        for (;;) {
            int u = 0;
            if (lane == 0) u = atomicAdd(&s_next, 1);
            u = __shfl_sync(0xffffffffu, u, 0);
            const long long item = lo + u;
            if (item >= hi) break;
            const int e = (int)(item / C::NU);
            const double *M = args.metric + (long long)e * C::NF * C::L3;
            double *__restrict__ outE = args.out + (long long)e * args.P;
            const int epar = (int)((reinterpret_cast<size_t>(outE) >> 3) & 1);
            v3_run_unit<S, P, L>((int)(item - (long long)e * C::NU), args, sT, W, M, outE, epar, buf, keep);
        }
    } else if (HXG_V3_FLOW && !C::FUSED && args.split == 1) {
        // one CTA counter over (element, unit) pairs: a warp that finds no unit left in
        // its element moves on to the CTA's next element instead of waiting at a barrier
        // for the element's last unit (8.6 % of the warp samples at H1 p5)
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        const long long nit = args.E > (int)blockIdx.x ? (args.E - 1 - (long long)blockIdx.x) / gridDim.x + 1 : 0;
        for (;;) {
            int u = 0;
            if (lane == 0) u = atomicAdd(&s_next, 1);
            u = __shfl_sync(0xffffffffu, u, 0);
            const int it = u / C::NU;
            if (it >= nit) break;
            const int e = (int)(blockIdx.x + (long long)it * gridDim.x);
            const double *M = args.metric + (long long)e * C::NF * C::L3;
            double *__restrict__ outE = args.out + (long long)e * args.P;
            const int epar = (int)((reinterpret_cast<size_t>(outE) >> 3) & 1);
            v3_run_unit<S, P, L>(u - it * C::NU, args, sT, W, M, outE, epar, buf, keep);
        }
    } else
    // persistent CTAs: work items (element, part) strided over the grid
    for (long long item = blockIdx.x; item < (long long)args.E * args.split; item += gridDim.x) {
    const int e = (int)(item / args.split);
    const int part = (int)(item - (long long)e * args.split);
    __syncthreads();  // previous item: every warp has left its unit loop
    if (threadIdx.x == 0) s_next = 0;
    const double *M;
    if constexpr (C::FUSED) {  // metric fields of this element (metric_kernel's body)
        double *sM = smem + C::OFF_M;
        const double *par = args.params + 24LL * e;
        const int knd = args.kind[e];
        const double cf = args.coef ? args.coef[e] : 1.0;
        for (int pt = threadIdx.x; pt < C::L3; pt += V3_THREADS) {
            const int n = pt / (L * L), l = (pt / L) % L, m = pt % L;
            double J[3][3], D[6], Cm[6], f[MAXF];
            dev_jacobian(knd, par, args.tables[TAB_NODES + l], args.tables[TAB_NODES + m],
                         args.tables[TAB_NODES + n], J);
            const double det = dev_metrics(J, D, Cm);
            const double w = args.tables[TAB_WTS + l] * args.tables[TAB_WTS + m] * args.tables[TAB_WTS + n];
            const double c = args.wgrid ? args.wgrid[(long long)e * C::L3 + (l * L + m) * L + n] : cf;
            dev_fields(S, det, D, Cm, w, c, f);
#pragma unroll
            for (int k = 0; k < C::NF; ++k) sM[k * C::L3 + pt] = f[k];
            if (!(det > 0.0) && part == 0) atomicOr(args.status + e, 1);
        }
        M = sM;
    } else {
#ifdef HXG_V3_FAKE_M  // timing experiment only: every element reads element 0's metric
        M = args.metric;
#else
        M = args.metric + (long long)e * C::NF * C::L3;
#endif
    }
    __syncthreads();
    double *__restrict__ outE = args.out + (long long)e * args.P;
    const int epar = (int)((reinterpret_cast<size_t>(outE) >> 3) & 1);
    const int lo = (int)((long long)C::NU * part / args.split);
    const int hi = (int)((long long)C::NU * (part + 1) / args.split);
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&s_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0) + lo;
        if (u >= hi) break;
        v3_run_unit<S, P, L>(u, args, sT, W, M, outE, epar, buf, keep);
    }
    }  // item loop
    if (args.E < 0 && keep == 0x9e3779b9u) args.out[0] = keep;  // never taken; keeps `keep` live
    bulk_wait_all();
}

}  // namespace hxg
