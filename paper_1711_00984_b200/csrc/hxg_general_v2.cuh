// hxg_general_v2.cuh -- compile-time specialized general-map Gram kernel.
//
// Same three-stage sum factorization as general_kernel (hxg_kernels.cuh), with
// the space, the (isotropic) order p and the rule size L as template
// parameters, so every extent, term list, group list and index division is a
// compile-time constant and all stage loops unroll.  One CTA integrates one
// work unit (element e, trial block b, test block a >= b, trial digit j3): the
// block-(a) columns of the packed rows J = (j1, j2, j3, b).
//
// Stage C (contraction over xi1) runs on FP64 DMMA (mma.sync m8n8k4) in one of
// two factorizations, chosen per block pair at compile time by FP64-pipe cost
// (DMMA and DFMA share the FP64 pipe on B200; profiles/peaks_r01.jsonl):
//   B-form: D[j1, (i1,i2,i3)] = sum_{h,l} u_s(j1,l) * (u_r(i1,l) B_h[i2,i3,l])
//           A operand = trial 1D table (registers), B operand = table x B_h
//   Y-form: D[j1, i1] (per (i2,i3)) = sum_{r,l} Y_r[j1,l] u_r(i1,l),
//           Y_r[j1,l] = sum_{h: r(h)=r} u_s(h)(j1,l) B_h[l]  (built per fragment)
//   P-form: D[(j2,i3,i2), (j1,i1)] = sum_{h,l} B_h[j2,i3,i2,l] * (u_s(j1,l) u_r(i1,l))
//           rows and columns both flattened: no digit padding of the 8x8 tiles,
//           B operand in registers, scattered staging stores (B-form pads j1 to
//           a multiple of 8: 56-69% tile occupancy at digit extents 9-11)
// The Y-form needs about nr*L FMAs per Gram entry instead of nh*L (H1: 2L vs
// 4L), at the price of 8x8 output tiles that span only n1a x n1b entries.
// Stage B (contraction over xi2) runs on DMMA as well when its tiles are dense
// enough (stageb_dmma), on DFMA otherwise.
#pragma once
#include "hxg_common.cuh"
#include "hxg_terms.h"

namespace hxg {

struct V2Args {
    const double *tables;  // TAB_TOTAL
    const double *metric;  // [E][nfields][n][l][m]
    double *out;           // [E][P]
    long long P;
    int E;
    // inputs of the fused low-order path (metric == NULL): see V3Cfg::FUSED
    const int *kind = nullptr;
    const double *params = nullptr, *coef = nullptr, *wgrid = nullptr;
    int *status = nullptr;
};

#ifndef HXG_V2_WARPS
#define HXG_V2_WARPS 8
#endif
#ifndef HXG_V2_BUDGET_KB
#define HXG_V2_BUDGET_KB 110
#endif
constexpr int V2_WARPS = HXG_V2_WARPS;
constexpr int V2_THREADS = V2_WARPS * 32;

#ifndef HXG_V2_STAGEB_EFF
#define HXG_V2_STAGEB_EFF 0.5
#endif

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int S, int P, int L>
struct V2Cfg {
    static constexpr int NB = nb_of(S);
    static constexpr int LP = (L + 1) & ~1;
    static constexpr int NF = nf_of(S);
    static constexpr int L3 = L * L * L;
    __host__ __device__ static constexpr int n(int a, int d) { return ext_of(S, P, a, d); }
    __host__ __device__ static constexpr int nmax(int d)
    {
        return cmax(n(0, d), NB > 1 ? cmax(n(1, d), n(2, d)) : 0);
    }
    __host__ __device__ static constexpr int off(int a)
    {
        return a == 0 ? 0 : (a == 1 ? n(0, 0) * n(0, 1) * n(0, 2)
                                    : n(0, 0) * n(0, 1) * n(0, 2) + n(1, 0) * n(1, 1) * n(1, 2));
    }
    static constexpr int N = off(NB - 1) + n(NB - 1, 0) * n(NB - 1, 1) * n(NB - 1, 2);
    static constexpr int N1 = nmax(0), N2 = nmax(1), N3 = nmax(2);
    __host__ __device__ static constexpr int c12(int a) { return n(a, 0) * n(a, 1); }
    static constexpr int C12 = cmax(c12(0), NB > 1 ? cmax(c12(1), c12(2)) : 0);
    __host__ __device__ static constexpr int maxg()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b < NB; ++b) m = cmax(m, make_pair_plan(S, a, b).ng);
        return m;
    }
    __host__ __device__ static constexpr int maxh()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b < NB; ++b) m = cmax(m, make_pair_plan(S, a, b).nh);
        return m;
    }
    static constexpr int NG = maxg(), NH = maxh();
    static constexpr int BUDGET = (HXG_V2_BUDGET_KB * 1024) / 8;  // doubles (110 KB: 2 CTAs per SM)
    __host__ __device__ static constexpr int sld(int R3) { return ((C12 * R3 + 7) / 8) * 8 + 2; }
    __host__ __device__ static constexpr int smem(int R2, int R3)
    {
        return 2 * KT * LP + R3 * NG * L * LP + R2 * NH * R3 * N2 * LP + R2 * N1 * sld(R3) + (R2 * N1 + 1) / 2;
    }
    __host__ __device__ static constexpr int pick_r3()
    {
        for (int r = N3; r >= 1; --r)
            if (smem(N2, r) <= BUDGET) return r;
        return 1;
    }
    static constexpr int R3 = pick_r3();
    __host__ __device__ static constexpr int pick_r2()
    {
        for (int r = N2; r >= 1; --r)
            if (smem(r, R3) <= BUDGET) return r;
        return 1;
    }
    static constexpr int R2 = pick_r2();
    static constexpr int SLD = sld(R3);
    static constexpr int OFF_T = 0;
    static constexpr int OFF_A = OFF_T + 2 * KT * LP;
    static constexpr int OFF_B = OFF_A + R3 * NG * L * LP;
    static constexpr int OFF_S = OFF_B + R2 * NH * R3 * N2 * LP;
    static constexpr int OFF_R = OFF_S + R2 * N1 * SLD;  // int[R2 * N1]: staging row offsets
    static constexpr int SMEM_BYTES = smem(R2, R3) * 8;
    static constexpr int SJ2 = NH * R3 * N2 * LP;  // sB stride per j2
    static constexpr int SH = R3 * N2 * LP;        // sB stride per h
    __host__ __device__ static constexpr int units()
    {
        int u = 0;
        for (int b = 0; b < NB; ++b) u += (NB - b) * n(b, 2);
        return u;
    }
    static constexpr int NU = units();
    static constexpr int MINB = SMEM_BYTES <= 113 * 1024 ? 2 : 1;

    // stage B on DMMA when the 8x8x4 tiles are not mostly padding: columns l pad to
    // 8, the contraction over m pads to 4 (rows run over the flattened (j2, i2) index)
    __host__ __device__ static constexpr bool stageb_dmma()
    {
        return (double)L / (8 * ((L + 7) / 8)) * (double)L / (4 * ((L + 3) / 4)) >= HXG_V2_STAGEB_EFF;
    }

    // stage-C factorization per block pair (see file header)
    __host__ __device__ static constexpr int yq(int a, int b)  // max #h sharing one test function
    {
        const CPair pp = make_pair_plan(S, a, b);
        int q = 1;
        for (int r = 0; r < pp.nr; ++r) {
            int hr = 0;
            for (int h = 0; h < pp.nh; ++h) hr += pp.h_r[h] == r;
            q = cmax(q, hr);
        }
        return q;
    }
    __host__ __device__ static constexpr bool yform(int a, int b)
    {
        const CPair pp = make_pair_plan(S, a, b);
        if (n(a, 0) > 8 || n(b, 0) > 8) return false;
        const int costB8 = n(a, 0) * ((pp.nh * L + 3) / 4) * 288;
        const int costY8 = 8 * ((pp.nr * L + 3) / 4) * (256 + 32 * yq(a, b));
        return costY8 < costB8;
    }
};

__device__ __forceinline__ void st_cs(double *p, double v) { __stcs(p, v); }

// bulk (TMA-engine) copy shared -> global, 16-byte aligned, size multiple of 16
// The Gram output is written once and never re-read by the kernel: mark it
// evict-first in L2 so the stream does not push the (re-read) metric fields
// out to DRAM.
#ifndef HXG_BULK_HINT
#define HXG_BULK_HINT 1
#endif
__device__ __forceinline__ void bulk_s2g(double *gdst, const double *ssrc, int bytes)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
#if HXG_BULK_HINT
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));  // not volatile: hoisted out of copy loops
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(gdst),
                 "r"(s), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// timing-only switches (wrong results): bit 0 skips stage A, 1 stage B, 2 the
// stage-C DMMAs, 3 the bulk write-out
#ifndef HXG_V2_SKIP
#define HXG_V2_SKIP 0
#endif
#ifndef HXG_V2_STAGEB_DMMA
#define HXG_V2_STAGEB_DMMA 1
#endif
#ifndef HXG_V2_PFORM
#define HXG_V2_PFORM 1
#endif
#ifndef HXG_V2_EVEN_CHUNKS
#define HXG_V2_EVEN_CHUNKS 1
#endif
#ifndef HXG_V2_AREG
#define HXG_V2_AREG 1
#endif
#ifndef HXG_V2_PF_RT
#define HXG_V2_PF_RT 2
#endif
#ifndef HXG_V2_PF_MINNH
#define HXG_V2_PF_MINNH 3
#endif
// B-form: trial rows j1 beyond the last full 8-row tile on DFMA instead of a
// mostly-empty DMMA row tile (both share the FP64 pipe), for at most HXG_V2_DREM
// such rows.  Measured (H(div), 1024 elements): 1 row (p = 8) +4 %, 2 rows (p = 9)
// -7 %, 3 rows (p = 10) -16 % -- the per-k-step shared-memory loads of the DFMA rows
// cost more than the DMMA padding they save beyond one row.
#ifndef HXG_V2_DREM
#define HXG_V2_DREM 1
#endif

template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void v2_process(const V2Args &args, double *smem, int e, int j3)
{
    using C = V2Cfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int LP = C::LP, L3 = C::L3, NG = C::NG, N2 = C::N2, R2 = C::R2, R3 = C::R3;
    constexpr int SLD = C::SLD, SJ2 = C::SJ2, SH = C::SH, N = C::N;
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n3a = C::n(A, 2);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha0 = sh_of(S, A, 0), sha1 = sh_of(S, A, 1), sha2 = sh_of(S, A, 2);
    constexpr int shb0 = sh_of(S, B, 0), shb1 = sh_of(S, B, 1), shb2 = sh_of(S, B, 2);
    constexpr int offA = C::off(A), offB = C::off(B);
    constexpr bool YF = C::yform(A, B);
    // product form instead of the B-form when the contraction is long enough (nh >= 3:
    // H1, H(curl)) to amortize its scattered staging stores; measured on p = 8..10
    constexpr bool PF = !YF && HXG_V2_PFORM && pp.nh >= HXG_V2_PF_MINNH;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    const double *sT = smem + C::OFF_T;
    double *sA = smem + C::OFF_A;
    double *sB = smem + C::OFF_B;
    double *sS = smem + C::OFF_S;
    int *sRow = reinterpret_cast<int *>(smem + C::OFF_R);
    const double *__restrict__ M = args.metric + (long long)e * C::NF * L3;
    double *__restrict__ outE = args.out + (long long)e * args.P;

    // ---- per-CTA stage-C operand registers ---------------------------------
    constexpr int KD = pp.nh * L;
    constexpr int NKS = (KD + 3) / 4;          // B-form k-steps
    constexpr int NMT0 = (n1b + 7) / 8;        // B-form row tiles
    constexpr int NREM = n1b % 8;              // rows of a partial last row tile
    constexpr bool DREM = NMT0 > 1 && NREM > 0 && NREM <= HXG_V2_DREM;
    constexpr int NMT = DREM ? NMT0 - 1 : NMT0;  // row tiles on DMMA
    constexpr int YQ = C::yq(A, B);            // Y-form trial factors per test function
    constexpr int KSY = (pp.nr * L + 3) / 4;   // Y-form k-steps (segments may straddle)
    constexpr int NKR = (YF || PF) ? 1 : NKS;  // register array extents
    constexpr int NYR = YF ? KSY : 1;
    double Af[NMT][NKR];
    int Ao[DREM ? NKR : 1];  // sT offset of u_s(j1 = 0 + shb0, l(k)) for the DFMA rows
    (void)Ao;
    double Yb[NYR];
    double Yc[NYR][YQ];
    int Yo[NYR][YQ];
    (void)Af; (void)Yb; (void)Yc; (void)Yo;
    if constexpr (PF) {
    } else if constexpr (!YF) {
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
            for (int ks = 0; ks < NKS; ++ks) {
                const int j1 = mt * 8 + g8, k = ks * 4 + t4;
                const int h = k / L, l = k - h * L;
                int fs = 0;
#pragma unroll
                for (int hh = 0; hh < pp.nh; ++hh)
                    if (hh == h) fs = pp.h_fs[hh];
                Af[mt][ks] = (k < KD && j1 < n1b) ? sT[(fs * KT + j1 + shb0) * LP + l] : 0.0;
                if constexpr (DREM) {
                    if (mt == 0) Ao[ks] = k < KD ? (fs * KT + shb0) * LP + l : -1;
                }
            }
    } else {
        // k = r L + l; lane t4 of k-step ks carries k = 4 ks + t4
#pragma unroll
        for (int ks = 0; ks < KSY; ++ks) {
            const int k = ks * 4 + t4;
            const bool kv = k < pp.nr * L;
            const int r = kv ? k / L : 0, l = kv ? k - (k / L) * L : 0;
            int rc = 0;
#pragma unroll
            for (int rr = 0; rr < pp.nr; ++rr)
                if (rr == r) rc = pp.r_code[rr];
            Yb[ks] = (kv && g8 < n1a) ? sT[(rc * KT + g8 + sha0) * LP + l] : 0.0;
#pragma unroll
            for (int q = 0; q < YQ; ++q) {
                Yc[ks][q] = 0.0;
                Yo[ks][q] = l;
            }
            int q = 0;
#pragma unroll
            for (int h = 0; h < pp.nh; ++h) {
                const bool mine = kv && pp.h_r[h] == r;
#pragma unroll
                for (int qq = 0; qq < YQ; ++qq)
                    if (mine && q == qq) {
                        Yc[ks][qq] = g8 < n1b ? sT[(pp.h_fs[h] * KT + g8 + shb0) * LP + l] : 0.0;
                        Yo[ks][qq] = h * SH + l;
                    }
                q += mine ? 1 : 0;
            }
        }
    }
    const int epar = (int)((reinterpret_cast<size_t>(outE) >> 3) & 1);

    // Stage A with the metric in registers: when every group is one term and one
    // pass of the CTA covers all (g, l, m) items (H(div), L2 at p >= 8), each
    // thread loads its L metric values once per unit instead of once per i3 (the
    // values do not depend on i3; the reload latency sat on a CTA barrier)
    constexpr bool AREG = R3 == 1 && pp.nt == pp.ng && pp.ng * L * L <= V2_THREADS && HXG_V2_AREG;
    double mv[AREG ? L : 1];
    (void)mv;
    if constexpr (AREG) {
        const int g = tid / (L * L), lm = tid - g * (L * L);
        int fld = 0;
#pragma unroll
        for (int t = 0; t < pp.nt; ++t)
            if (pp.t_g[t] == g) fld = pp.t_field[t];
        const bool v = tid < pp.ng * L * L;
#pragma unroll
        for (int n = 0; n < L; ++n) mv[n] = v ? __ldg(M + fld * L3 + n * L * L + lm) : 0.0;
    }

    const int i3first = (A == B) ? j3 : 0;
    for (int i3lo = i3first; i3lo < n3a; i3lo += R3) {
        const int r3 = cmin(R3, n3a - i3lo);
        const int ncols = n1a * n2a * r3;
        __syncthreads();
        // ---------------- stage A: contract xi3 -> Abar_g[ii3][g][m][l] ----------------
        if constexpr (AREG) {
            if (tid < pp.ng * L * L && !(HXG_V2_SKIP & 1)) {
                const int g = tid / (L * L), lm = tid - g * (L * L);
                const int i3 = i3lo;
                double s = 0.0;
#pragma unroll
                for (int t = 0; t < pp.nt; ++t) {
                    if (pp.t_g[t] != g) continue;
                    const double *Ta = sT + (pp.t_fr[t] * KT + i3 + sha2) * LP;
                    const double *Tb = sT + (pp.t_fs[t] * KT + j3 + shb2) * LP;
#pragma unroll
                    for (int n = 0; n < L; ++n) s = fma(mv[n], Ta[n] * Tb[n], s);
                    if (pp.t_sign[t] < 0) s = -s;
                }
                const int l = lm / L, m = lm - l * L;
                sA[(g * L + m) * LP + l] = s;
            }
        } else
        // (g, ii3, l, m) items over all threads (the group index is a runtime value)
        for (int it2 = tid; it2 < (HXG_V2_SKIP & 1 ? 0 : pp.ng * r3 * L * L); it2 += V2_THREADS) {
            const int g = it2 / (r3 * L * L), it = it2 - g * (r3 * L * L);
            {
                const int ii3 = it / (L * L), lm = it - ii3 * (L * L);
                const int i3 = i3lo + ii3;
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < pp.nt; ++t) {
                    if (pp.t_g[t] != g) continue;
                    const double *Mf = M + pp.t_field[t] * L3 + lm;
                    const double *Ta = sT + (pp.t_fr[t] * KT + i3 + sha2) * LP;
                    const double *Tb = sT + (pp.t_fs[t] * KT + j3 + shb2) * LP;
                    double s = 0.0;
#pragma unroll
                    for (int n = 0; n < L; ++n) s = fma(__ldg(Mf + n * L * L), Ta[n] * Tb[n], s);
                    acc += pp.t_sign[t] > 0 ? s : -s;
                }
                const int l = lm / L, m = lm - l * L;
                sA[((ii3 * NG + g) * L + m) * LP + l] = acc;
            }
        }
        // j2 chunks of equal size (n2b = 11, R2 = 8 -> 6 + 5 rather than 8 + 3)
        constexpr int NCH = (n2b + R2 - 1) / R2, R2E = HXG_V2_EVEN_CHUNKS ? (n2b + NCH - 1) / NCH : R2;
        for (int j2lo = 0; j2lo < n2b; j2lo += R2E) {
            const int r2 = cmin(R2E, n2b - j2lo);
            if (j2lo == 0) __syncthreads();  // stage A (sA) complete; later chunks: the
                                             // barrier before the write-out already orders
                                             // stage C reads of sB before its next writes
            // ---------------- stage B: contract xi2 -> B_h[jj2][h][ii3][i2][l] ----------------
#if HXG_V2_STAGEB_DMMA
            // on DMMA: B_h[(jj2,i2)][l] = sum_{g in h} sum_m V_g[(jj2,i2)][m] Abar_g[m][l] with
            // V_g = u_fr(i2,m) u_fs(j2,m); tile rows run over the flattened (jj2, i2) index,
            // one warp per (h, ii3, 8-row tile), all l tiles in flight
            if constexpr (C::stageb_dmma()) {
                constexpr int NLT = (L + 7) / 8, LQ = (L + 3) / 4;
                const int nrt = (r2 * n2a + 7) >> 3;
                for (int w = warp; w < (HXG_V2_SKIP & 2 ? 0 : pp.nh * r3 * nrt); w += V2_WARPS) {
                    __syncwarp();  // converged for mma.sync (.aligned) after divergent code
                    const int h = w / (r3 * nrt), w2 = w - h * (r3 * nrt);
                    const int ii3 = w2 / nrt, rt = w2 - ii3 * nrt;
                    const int row = rt * 8 + g8;
                    const bool rv = row < r2 * n2a;
                    const int jj2 = rv ? row / n2a : 0, i2 = rv ? row - jj2 * n2a : 0;
                    const int j2 = j2lo + jj2;
                    double d[NLT][2];
#pragma unroll
                    for (int lt = 0; lt < NLT; ++lt) d[lt][0] = d[lt][1] = 0.0;
#pragma unroll
                    for (int g = 0; g < pp.ng; ++g) {
                        if (pp.g_h[g] != h) continue;
                        const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sha1) * LP;
                        const double *Tb = sT + (pp.g_fs[g] * KT + j2 + shb1) * LP;
                        const double *Ag = sA + (ii3 * NG + g) * L * LP;
#pragma unroll
                        for (int ks = 0; ks < LQ; ++ks) {
                            const int m = ks * 4 + t4;
                            const double av = (m < L && rv) ? Ta[m] * Tb[m] : 0.0;
#pragma unroll
                            for (int lt = 0; lt < NLT; ++lt) {
                                const double bv = m < L ? Ag[m * LP + lt * 8 + g8] : 0.0;
                                dmma_8x8x4(d[lt][0], d[lt][1], av, bv);
                            }
                        }
                    }
                    if (rv) {
                        double *dst = sB + jj2 * SJ2 + ((h * R3 + ii3) * N2 + i2) * LP;
#pragma unroll
                        for (int lt = 0; lt < NLT; ++lt) {
                            const int l = lt * 8 + 2 * t4;
                            if (l < L) dst[l] = d[lt][0];
                            if (l + 1 < L) dst[l + 1] = d[lt][1];
                        }
                    }
                }
            } else
#endif
            // (h, jj2, ii3, i2) items over all threads
            for (int it2 = tid; it2 < (HXG_V2_SKIP & 2 ? 0 : pp.nh * R2 * R3 * n2a); it2 += V2_THREADS) {
                const int h = it2 / (R2 * R3 * n2a), it = it2 - h * (R2 * R3 * n2a);
                {
                    const int i2 = it % n2a, q = it / n2a, ii3 = q % R3, jj2 = q / R3;
                    if (ii3 >= r3 || jj2 >= r2) continue;
                    const int j2 = j2lo + jj2;
                    double acc[LP];
#pragma unroll
                    for (int l = 0; l < LP; ++l) acc[l] = 0.0;
#pragma unroll
                    for (int g = 0; g < pp.ng; ++g) {
                        if (pp.g_h[g] != h) continue;
                        const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sha1) * LP;
                        const double *Tb = sT + (pp.g_fs[g] * KT + j2 + shb1) * LP;
                        const double *Ag = sA + (ii3 * NG + g) * L * LP;
#pragma unroll
                        for (int m = 0; m < L; ++m) {
                            const double v = Ta[m] * Tb[m];
                            const double2 *Am = reinterpret_cast<const double2 *>(Ag + m * LP);
#pragma unroll
                            for (int l2 = 0; l2 < LP / 2; ++l2) {
                                const double2 av = Am[l2];
                                acc[2 * l2] = fma(av.x, v, acc[2 * l2]);
                                acc[2 * l2 + 1] = fma(av.y, v, acc[2 * l2 + 1]);
                            }
                        }
                    }
                    double2 *dst = reinterpret_cast<double2 *>(sB + jj2 * SJ2 + ((h * R3 + ii3) * N2 + i2) * LP);
#pragma unroll
                    for (int l2 = 0; l2 < LP / 2; ++l2) dst[l2] = make_double2(acc[2 * l2], acc[2 * l2 + 1]);
                }
            }
            // staging row `row` = (jj2, j1) is shifted by pad(row) in {0,1} doubles so that
            // it has the 16-byte phase of its global destination (bulk-copy alignment)
            const int I0 = offA + n1a * n2a * i3lo;
            auto row_goff = [&](int jj2, int j1) {
                const int J = offB + j1 + n1b * (j2lo + jj2 + n2b * j3);
                return J * N - J * (J - 1) / 2 - J + I0;  // &G(J, I0) - outE
            };
            for (int row = tid; row < r2 * n1b; row += V2_THREADS) {
                const int jj2 = row / n1b, j1 = row - jj2 * n1b;
                sRow[row] = row * SLD + ((epar + row_goff(jj2, j1)) & 1);
            }
            bulk_wait_read();  // previous chunk's bulk stores have read the staging buffer
            __syncthreads();
            // ---------------- stage C: contract xi1 on DMMA ----------------
            if constexpr (PF) {
                // product form: G[(jj2,ii3,i2), (j1,i1)] = sum_{h,l} B_h[jj2][ii3][i2][l] * [u_s(j1,l) u_r(i1,l)]
                // Tile rows (jj2, ii3, i2) and columns (j1, i1) are both flattened, so the
                // 8x8 tiles carry no digit padding (the B-form pads j1 to 8 or 16).  The B
                // operand (a product of two 1D tables) stays in registers while a warp
                // sweeps the row tiles of one column tile, two row tiles in flight.
                // columns (j1, i1) with i1 padded to an even count, so a lane's two output
                // columns (2 t4, 2 t4 + 1) share j1 and sit next to each other in staging
                constexpr int N1E = (n1a + 1) & ~1, NCOL = n1b * N1E, NCT = (NCOL + 7) / 8;
                const int nrow = r2 * r3 * n2a, nrt = (nrow + 7) >> 3;
                constexpr int RT = HXG_V2_PF_RT;  // row tiles in flight per warp
                const int nrtp = (nrt + RT - 1) / RT;  // row-tile groups per column tile
                const int T = NCT * nrtp;
                const int per = (T + V2_WARPS - 1) / V2_WARPS;
                const int it0 = warp * per, it1 = cmin(T, it0 + per);
                double Bp[NKS];
                int ko[NKS];
                int ctc = -1, dj1 = -1, di1 = 0;
                for (int it = it0; it < it1; ++it) {
                    __syncwarp();  // converged for mma.sync (.aligned) after divergent code
                    const int ct = it / nrtp, rt0 = RT * (it - ct * nrtp);
                    if (ct != ctc) {  // (re)load the B fragment of column tile ct
                        ctc = ct;
                        const int col = ct * 8 + g8;
                        const int j1 = col / N1E, i1 = col - j1 * N1E;
                        const bool cv = col < NCOL && i1 < n1a;
#pragma unroll
                        for (int ks = 0; ks < NKS; ++ks) {
                            const int k = ks * 4 + t4;
                            const int h = k / L, l = k - h * L;
                            int fs = 0, fr = 0;
#pragma unroll
                            for (int hh = 0; hh < pp.nh; ++hh)
                                if (hh == h) { fs = pp.h_fs[hh]; fr = pp.h_fr[hh]; }
                            const bool v = k < KD;
                            Bp[ks] = (v && cv) ? sT[(fs * KT + j1 + shb0) * LP + l] * sT[(fr * KT + i1 + sha0) * LP + l]
                                               : 0.0;
                            ko[ks] = v ? h * SH + l : 0;
                        }
                        {  // output columns 2 t4, 2 t4 + 1 of this lane
                            const int oc = ct * 8 + 2 * t4;
                            dj1 = oc < NCOL ? oc / N1E : -1;
                            di1 = oc - (oc / N1E) * N1E;
                        }
                    }
                    double d[RT][2];
#pragma unroll
                    for (int c = 0; c < RT; ++c) d[c][0] = d[c][1] = 0.0;
                    int ao[RT], jr[RT], sc[RT];
#pragma unroll
                    for (int c = 0; c < RT; ++c) {  // this lane's row g8 of row tile rt0 + c
                        const int row = (rt0 + c) * 8 + g8;
                        const bool rv = row < nrow;
                        const int i2 = rv ? row % n2a : 0, q = rv ? row / n2a : 0;
                        const int ii3 = R3 == 1 ? 0 : q % r3, jj2 = R3 == 1 ? q : q / r3;
                        ao[c] = rv ? jj2 * SJ2 + (ii3 * N2 + i2) * LP : 0;
                        jr[c] = rv ? jj2 * n1b : -1;
                        sc[c] = (ii3 * n2a + i2) * n1a;
                    }
#pragma unroll
                    for (int ks = 0; ks < (HXG_V2_SKIP & 4 ? 0 : NKS); ++ks) {
#pragma unroll
                        for (int c = 0; c < RT; ++c) dmma_8x8x4(d[c][0], d[c][1], sB[ao[c] + ko[ks]], Bp[ks]);
                    }
                    if (dj1 >= 0 && !(HXG_V2_SKIP & 16)) {
#pragma unroll
                        for (int c = 0; c < RT; ++c) {
                            if (jr[c] < 0) continue;
                            double *dst = sS + sRow[jr[c] + dj1] + sc[c] + di1;
                            dst[0] = d[c][0];
                            if (di1 + 1 < n1a) dst[1] = d[c][1];
                        }
                    }
                }
            } else if constexpr (!YF) {
                const int nct = (ncols + 7) >> 3;
                const int T = nct * r2;
                const int per = (T + V2_WARPS - 1) / V2_WARPS;
                const int it0 = warp * per, it1 = cmin(T, it0 + per);
                int ct = -1;
                double X[NKS];
                int bo[NKS];
                int ctn = it0 / r2, jj2 = it0 - ctn * r2;  // tiles (ct, jj2), jj2 fastest
                for (int it = it0; it < it1; ++it) {
                    __syncwarp();  // converged for mma.sync (.aligned) after divergent code
                    if (ctn != ct) {
                        ct = ctn;
                        const int c = ct * 8 + g8;
                        const bool cval = c < ncols;
                        const int i1 = c % n1a, q = c / n1a, i2 = q % n2a, ii3 = q / n2a;
#pragma unroll
                        for (int ks = 0; ks < NKS; ++ks) {
                            const int k = ks * 4 + t4;
                            const int h = k / L, l = k - h * L;
                            int fr = 0;
#pragma unroll
                            for (int hh = 0; hh < pp.nh; ++hh)
                                if (hh == h) fr = pp.h_fr[hh];
                            const bool v = k < KD && cval;
                            X[ks] = v ? sT[(fr * KT + i1 + sha0) * LP + l] : 0.0;
                            bo[ks] = v ? (h * SH + (ii3 * N2 + i2) * LP + l) : 0;
                        }
                    }
                    const double *sBj = sB + jj2 * SJ2;
                    double d[NMT][2];
#pragma unroll
                    for (int mt = 0; mt < NMT; ++mt) d[mt][0] = d[mt][1] = 0.0;
                    double pr[DREM ? NREM : 1];  // DFMA rows j1 = 8 NMT + r, column ct 8 + g8
#pragma unroll
                    for (int r = 0; r < (DREM ? NREM : 1); ++r) pr[r] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < (HXG_V2_SKIP & 4 ? 0 : NKS); ++ks) {
                        const double bv = X[ks] * sBj[bo[ks]];
#pragma unroll
                        for (int mt = 0; mt < NMT; ++mt) dmma_8x8x4(d[mt][0], d[mt][1], Af[mt][ks], bv);
                        if constexpr (DREM) {
                            if (Ao[ks] >= 0) {
#pragma unroll
                                for (int r = 0; r < NREM; ++r) pr[r] = fma(sT[Ao[ks] + (8 * NMT + r) * LP], bv, pr[r]);
                            }
                        }
                    }
                    if constexpr (DREM) {  // sum the four k-lanes (t4) of each column g8
#pragma unroll
                        for (int r = 0; r < NREM; ++r) {
                            pr[r] += __shfl_xor_sync(0xffffffffu, pr[r], 1);
                            pr[r] += __shfl_xor_sync(0xffffffffu, pr[r], 2);
                        }
                        if (t4 < NREM) {  // lane t4 stores row 8 NMT + t4
                            double v = pr[0];
#pragma unroll
                            for (int r = 1; r < NREM; ++r)
                                if (t4 == r) v = pr[r];
                            sS[sRow[jj2 * n1b + 8 * NMT + t4] + ct * 8 + g8] = v;
                        }
                    }
#pragma unroll
                    for (int mt = 0; mt < NMT; ++mt) {
                        const int j1 = mt * 8 + g8;
                        if (j1 < n1b) {
                            double *dst = sS + sRow[jj2 * n1b + j1] + ct * 8 + 2 * t4;
                            dst[0] = d[mt][0];
                            dst[1] = d[mt][1];
                        }
                    }
                    if (++jj2 == r2) {
                        jj2 = 0;
                        ++ctn;
                    }
                }
            } else {
                const int T = r3 * n2a * r2;  // tiles (ii3, i2, jj2), jj2 fastest
                const int per = (T + V2_WARPS - 1) / V2_WARPS;
                const int it0 = warp * per, it1 = cmin(T, it0 + per);
                int qd = it0 / r2, jj2 = it0 - qd * r2;
                int ii3 = qd / n2a, i2 = qd - ii3 * n2a;
                for (int it = it0; it < it1; ++it) {
                    __syncwarp();  // converged for mma.sync (.aligned) after divergent code
                    const double *base = sB + jj2 * SJ2 + (ii3 * N2 + i2) * LP;
                    double d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int ks = 0; ks < KSY; ++ks) {
                        double y = Yc[ks][0] * base[Yo[ks][0]];
#pragma unroll
                        for (int q = 1; q < YQ; ++q) y = fma(Yc[ks][q], base[Yo[ks][q]], y);
                        dmma_8x8x4(d0, d1, y, Yb[ks]);
                    }
                    if (g8 < n1b) {
                        double *dst = sS + sRow[jj2 * n1b + g8] + (ii3 * n2a + i2) * n1a + 2 * t4;
                        if (2 * t4 < n1a) dst[0] = d0;
                        if (2 * t4 + 1 < n1a) dst[1] = d1;
                    }
                    if (++jj2 == r2) {
                        jj2 = 0;
                        if (++i2 == n2a) { i2 = 0; ++ii3; }
                    }
                }
            }
            fence_proxy_async();  // staging writes -> visible to the bulk-copy (async) proxy
            __syncthreads();
            // ---------------- write-out: one bulk copy per packed row segment ----------------
#ifdef HXG_V2_NO_BULK
            {  // warp per row, coalesced 8-byte stores (staging free at the next barrier)
                const int rows = r2 * n1b;
                for (int row = warp; row < rows; row += V2_WARPS) {
                    const int jj2 = row / n1b, j1 = row - jj2 * n1b;
                    const int goff = row_goff(jj2, j1);
                    const int J = offB + j1 + n1b * (j2lo + jj2 + n2b * j3);
                    const int cs = J > I0 ? J - I0 : 0;
                    const double *src = sS + row * SLD + ((epar + goff) & 1);
                    for (int c = cs + lane; c < ncols; c += 32) st_cs(outE + goff + c, src[c]);
                }
            }
            if (false)
#endif
            {
                const int rows = r2 * n1b;
                for (int row = tid; row < rows; row += V2_THREADS) {
                    const int jj2 = row / n1b, j1 = row - jj2 * n1b;
                    const int goff = row_goff(jj2, j1);
                    const int J = offB + j1 + n1b * (j2lo + jj2 + n2b * j3);
                    int cs = J > I0 ? J - I0 : 0;
                    if (cs >= ncols) continue;
                    const int pad = (epar + goff) & 1;
                    const double *src = sS + row * SLD + pad + cs;
                    double *dst = outE + goff + cs;
                    int len = ncols - cs;
                    if (reinterpret_cast<size_t>(dst) & 8) {  // 8-byte head
                        st_cs(dst, *src);
                        ++dst;
                        ++src;
                        --len;
                    }
                    if (len & 1) st_cs(dst + len - 1, src[len - 1]);  // 8-byte tail
                    if (len >= 2 && !(HXG_V2_SKIP & 8)) bulk_s2g(dst, src, (len & ~1) * 8);
                }
                bulk_commit();
            }
        }
    }
    bulk_wait_all();
}

template <int S, int P, int L>
__global__ void __launch_bounds__(V2_THREADS, (V2Cfg<S, P, L>::MINB))
    general_v2_kernel(const __grid_constant__ V2Args args)
{
    using C = V2Cfg<S, P, L>;
    extern __shared__ __align__(16) double smem[];
    const int u = blockIdx.x % C::NU;
    const int e = blockIdx.x / C::NU;
    // decode (b, a, j3): pairs enumerated b-major, a >= b
    int rem = u, pair = -1, j3 = 0;
#pragma unroll
    for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int a = b; a < C::NB; ++a) {
            if (pair < 0) {
                if (rem < C::n(b, 2)) { pair = a * 3 + b; j3 = rem; }
                else rem -= C::n(b, 2);
            }
        }
    double *sT = smem + C::OFF_T;
    for (int idx = threadIdx.x; idx < 2 * KT * C::LP; idx += V2_THREADS) {
        const int fk = idx / C::LP, l = idx - fk * C::LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    __syncthreads();
    if constexpr (C::NB == 1) {
        v2_process<S, P, L, 0, 0>(args, smem, e, j3);
    } else {
        switch (pair) {
        case 0: v2_process<S, P, L, 0, 0>(args, smem, e, j3); break;
        case 3: v2_process<S, P, L, 1, 0>(args, smem, e, j3); break;
        case 6: v2_process<S, P, L, 2, 0>(args, smem, e, j3); break;
        case 4: v2_process<S, P, L, 1, 1>(args, smem, e, j3); break;
        case 7: v2_process<S, P, L, 2, 1>(args, smem, e, j3); break;
        default: v2_process<S, P, L, 2, 2>(args, smem, e, j3); break;
        }
    }
}

}  // namespace hxg
