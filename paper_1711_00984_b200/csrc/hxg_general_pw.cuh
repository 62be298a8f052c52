// hxg_general_pw.cuh -- warp-owned product-form general-map Gram kernel for
// digit extents up to 12 and rules up to L = 12 (the default route for test
// orders p = 8..10; HXG_PW=1 also selects it at p = 4..7).
//
// Reference loops: tens_{h1,hcurl,hdiv,l2}_alt (_kernels.py:356-1150); the
// term / group model is hxg_plan.h.
//
// One warp owns a work unit (element e, trial block b, test block a >= b,
// digits j3, i3) and runs, with warp-private shared memory and no CTA barrier:
//   stage A (xi3, DFMA)  Abar_g[m][l] = sum_{t in g} sign_t sum_n M_t[n][l][m] u(i3,n) u(j3,n)
//   per group of NJ2 in {8, 4, 2, 1} trial digits j2 (rows r = i2 * NJ2 + jj2):
//     stage B (xi2, DMMA)  B_h[r][l] = sum_{g in h} sum_m V_g[r][m] Abar_g[m][l],
//                          V_g = u_fr(i2,m) u_fs(j2,m)
//     stage C (xi1, DMMA)  P-form: D[r, (j1,i1)] = sum_{(h,l)} B_h[r][l] * u_s(j1,l) u_r(i1,l)
//                          rows r and columns (j1,i1) flattened, K = (h,l) flattened: the
//                          8x8x4 tiles are padded only in the last tile of each dimension
//                          (the Y/B-forms of v2/v3 pad a digit extent of 9-11 to 16)
//     write-out            column tiles run in j1 order; when trial digit j1 is complete its
//                          NJ2 packed row segments (j1, j2), each n1a*n2a contiguous doubles,
//                          leave the j1's staging slot by one bulk copy (cp.async.bulk) each
// Rows interleave the group's trial digits (r = i2 * NJ2 + jj2, NJ2 | 8), so a lane's
// rows in every row tile share one jj2: the staging address of a D fragment is one
// per-(lane, column) base plus a compile-time row-tile stride.  Stage-C operands:
// A = B_h in fragment order in shared memory (conflict-free 8-byte loads, shared by
// CTW column tiles), B = two 1D-table loads and one DMUL per fragment, shared by the
// group's row tiles.
#pragma once
#include "hxg_common.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_terms.h"

namespace hxg {

#ifndef HXG_PW_WARPS
#define HXG_PW_WARPS 4
#endif
#ifndef HXG_PW_BUDGET_KB
#define HXG_PW_BUDGET_KB 112  // per CTA: 2 CTAs per SM
#endif
#ifndef HXG_PW_RJMAX
#define HXG_PW_RJMAX 8
#endif
// write-out: 1 = each D fragment value stored straight to HBM (8-byte streaming
// stores, no staging); 0 = staged per trial digit j1 in shared memory and written by
// bulk copies (cp.async.bulk) of whole packed row segments; -1 (default) = direct for
// the FP64-bound spaces H1 / H(curl) (few output bytes per flop: the scattered
// stores are absorbed), bulk for the HBM-bound H(div) / L2 (measured: the 8-byte
// stores leave 2.8x the output in L2 sector writes and stall on store back-pressure)
#ifndef HXG_PW_WO
#define HXG_PW_WO -1
#endif
__host__ __device__ constexpr bool pw_direct(int S) { return HXG_PW_WO < 0 ? (S == H1 || S == HCURL) : HXG_PW_WO == 1; }
// test digits i3 per work unit (stage-C rows (kk, i2) with kk < K; each packed row
// segment is K * n1a * n2a long, so the bulk write-out issues K times fewer copies
// per byte); default 1, HXG_PW_K_HDIV / HXG_PW_K_L2 for the staged spaces
#ifndef HXG_PW_K_HDIV
#define HXG_PW_K_HDIV 1
#endif
#ifndef HXG_PW_K_L2
#define HXG_PW_K_L2 1
#endif
#ifndef HXG_PW_STCS
#define HXG_PW_STCS 1  // direct write-out with evict-first streaming stores (else write-back)
#endif
#ifndef HXG_PW_CTW_NK
#define HXG_PW_CTW_NK 6  // two column tiles per step when the pair has <= this many k-steps
#endif
#ifndef HXG_PW_SKIP_WO
#define HXG_PW_SKIP_WO 0  // timing experiment only (wrong results): 1 no copy-out, 2 no staging either
#endif
// stage-C A operand (B_h fragments of the group's row tiles) held in registers for the
// whole group instead of re-read from shared memory at every column tile: -1 (default) =
// for the staged (HBM-bound) spaces, 0 never, 1 always
#ifndef HXG_PW_ASTAT
#define HXG_PW_ASTAT -1
#endif
#ifndef HXG_PW_STSWZ
#define HXG_PW_STSWZ 0  // staged write-out: swizzled store order (see pw_step)
#endif
// A-stationary groups: most stage-C A-fragment doubles a lane holds (row tiles x k-steps);
// block pairs whose 8-digit groups need more run 4-digit (2-, 1-digit) groups
#ifndef HXG_PW_AREG_MAX
#define HXG_PW_AREG_MAX 50
#endif
#ifndef HXG_PW_NSG_MAX
#define HXG_PW_NSG_MAX 0  // > 0: short groups re-divide the staging area into up to this many slots (measured: no gain)
#endif
#ifndef HXG_PW_BHOIST
#define HXG_PW_BHOIST 2  // stage-B B fragments (Abar) and trial-side 1D values in registers per group: 1 A-stationary groups only, 2 every group (direct spaces +0.2-3.5 % at p 8-10)
#endif
// direct spaces: block pairs whose group holds at most this many A-fragment doubles per lane
// also keep them in registers (0: never; measured -2 to -4 % for H(curl) p 8-10 at 24 / 40)
#ifndef HXG_PW_ASTAT_PAIR
#define HXG_PW_ASTAT_PAIR 0
#endif
__host__ __device__ constexpr bool pw_astat(int S) { return HXG_PW_ASTAT < 0 ? !pw_direct(S) : HXG_PW_ASTAT == 1; }
constexpr int PW_WARPS = HXG_PW_WARPS;
constexpr int PW_THREADS = PW_WARPS * 32;

template <int S, int P, int L>
struct PWCfg {
    using C2 = V2Cfg<S, P, L>;
    static constexpr int NB = C2::NB, NF = C2::NF, L3 = C2::L3, N = C2::N;
    static constexpr int NG = C2::NG, NH = C2::NH, C12 = C2::C12;
    __host__ __device__ static constexpr int n(int a, int d) { return C2::n(a, d); }
    static constexpr int LQ = (L + 3) / 4;       // k-steps of stage B (K = m)
    static constexpr int LT = (L + 7) / 8;       // column tiles of stage B (N = l)
    static constexpr int LP = cmax(12, 4 * LQ);  // sT row stride (zero padded beyond L)
    static constexpr bool OK = L <= 12 && C2::N1 <= 12 && C2::N2 <= 12 && C2::N3 <= 12;
    __host__ __device__ static constexpr int maxt()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b < NB; ++b) m = cmax(m, make_pair_plan(S, a, b).nt);
        return m;
    }
    static constexpr int NT = maxt();
    __host__ __device__ static constexpr int nk(int a, int b) { return (make_pair_plan(S, a, b).nh * L + 3) / 4; }
    // two column tiles per step only with the direct write-out: the staged spaces keep
    // one (fewer staging slots; measured faster at p = 9, 10)
    __host__ __device__ static constexpr int ctw(int a, int b)
    {
        return (pw_direct(S) && nk(a, b) <= HXG_PW_CTW_NK) ? 2 : 1;
    }
    __host__ __device__ static constexpr int maxnk()
    {
        int m = 1;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b <= a; ++b) m = cmax(m, nk(a, b));
        return m;
    }
    static constexpr int NKS = maxnk();
    static constexpr int K = S == HDIV ? HXG_PW_K_HDIV : (S == L2 ? HXG_PW_K_L2 : 1);
    __host__ __device__ static constexpr int kcnt(int r) { return (r + K - 1) / K; }  // units over r digits i3
    static constexpr int N2M = K * C2::N2;  // stage-C rows (kk, i2) per trial digit j2
    // most trial digits j1 beyond the first that one step (CTW 8-column tiles of
    // (j1, i1)) touches
    __host__ __device__ static constexpr int jspan()
    {
        int m = 0;
        for (int a = 0; a < NB; ++a)
            for (int b = 0; b <= a; ++b) {
                const int n1a = n(a, 0), ncol = n(b, 0) * n1a, w = 8 * ctw(a, b);
                for (int c0 = 0; c0 < ncol; c0 += w) m = cmax(m, cmin(c0 + w - 1, ncol - 1) / n1a - c0 / n1a);
            }
        return m;
    }
    static constexpr int JSPAN = jspan();
    // staging slots, one per trial digit j1 in flight: the JSPAN + 1 digits one step
    // writes plus one whose bulk copies may still be reading
    static constexpr int NSLOT = JSPAN + 2;
    static constexpr int NSLOT_SMEM = pw_direct(S) ? 0 : NSLOT;
    // a group of nj2 < RJ trial digits divides the same staging area into more, smaller
    // slots (nj2 segments each): short groups have short steps, and with NSLOT slots a
    // step would wait for the smem reads of the bulk copies issued two steps earlier
    __host__ __device__ static constexpr int nsg(int nj2, int rj)
    {
        return HXG_PW_NSG_MAX > 0 ? cmin(HXG_PW_NSG_MAX, (NSLOT * rj) / nj2) : NSLOT;
    }
    // segments per slot
    __host__ __device__ static constexpr int slotrows(int nj2, int rj) { return HXG_PW_NSG_MAX > 0 ? nj2 : rj; }
    static constexpr int WARPS = PW_WARPS, THREADS = PW_THREADS;
    static constexpr int SEG = ((K * C12 + 2 + 1) / 2) * 2;  // staging segment stride (even, >= K C12 + 1)
    // per-warp shared memory (doubles) for groups of at most rj in {1, 2, 4, 8} trial digits
    __host__ __device__ static constexpr int rtmax(int rj) { return K * ((rj * C2::N2 + 7) / 8); }
    __host__ __device__ static constexpr int w_tot(int rj)
    {
        return K * NT * LP + K * NG * LT * LQ * 32 + (pw_astat(S) ? 1 : rtmax(rj)) * NKS * 32 + NSLOT_SMEM * rj * SEG;
    }
    __host__ __device__ static constexpr int cta_bytes(int rj) { return (2 * KT * LP + WARPS * w_tot(rj)) * 8 + 16; }
    // RJCAP: optional cap on the trial digits per group (test hook; the round-2 H1 p = 7
    // failure of 8-digit groups was a missing warp reconvergence before mma.sync, fixed
    // by the __syncwarp() ahead of every DMMA block -- profiles/pw_h1p7_r02.txt)
#ifndef HXG_PW_RJCAP_H1
#define HXG_PW_RJCAP_H1 8
#endif
    static constexpr int RJCAP = S == H1 ? HXG_PW_RJCAP_H1 : 8;
    __host__ __device__ static constexpr int pick_rj()
    {
        int r = 1;
        for (int q = 2; q <= cmin(cmin(HXG_PW_RJMAX, RJCAP), 8); q *= 2)
            if (q / 2 < N2M && cta_bytes(q) <= HXG_PW_BUDGET_KB * 1024) r = q;
        return r;
    }
    static constexpr int RJ = pick_rj();
    static constexpr int RTM = rtmax(RJ);
    static constexpr int W_P = 0;                        // [NT][LP] stage-A 1D products
    static constexpr int W_A = W_P + K * NT * LP;            // [K][NG][LT][LQ][32] Abar (stage-B B fragments)
    static constexpr int W_B = W_A + K * NG * LT * LQ * 32;  // [RTM][NKS][32] B_h (stage-C A fragments)
    static constexpr int W_S = W_B + (pw_astat(S) ? 1 : RTM) * NKS * 32;  // [NSLOT][RJ][SEG] staging
    static constexpr int W_TOT = w_tot(RJ);
    static constexpr int OFF_T = 0;
    static constexpr int OFF_W = 2 * KT * LP;
    static constexpr int SMEM_BYTES = cta_bytes(RJ);
#ifndef HXG_PW_MAXB
#define HXG_PW_MAXB 2
#endif
    static constexpr int MINB = cmax(1, cmin(HXG_PW_MAXB, (228 * 1024) / (SMEM_BYTES + 1024)));
    __host__ __device__ static constexpr int units()
    {
        int u = 0;
        for (int b = 0; b < NB; ++b)
            for (int a = b; a < NB; ++a) {
                if (a == b)
                    for (int j3 = 0; j3 < n(b, 2); ++j3) u += kcnt(n(b, 2) - j3);
                else
                    u += n(b, 2) * kcnt(n(a, 2));
            }
        return u;
    }
    static constexpr int NU = units();
};

__host__ __device__ constexpr int pw_rj_cap(int K, int n2a, int nk)
{
    int r = 1;
    for (int q = 2; q <= 8; q *= 2)
        if (K * ((q * n2a + 7) / 8) * nk <= HXG_PW_AREG_MAX) r = q;
    return r;
}

template <int I>
struct PWInt {
    static constexpr int value = I;
};
template <int N, int I = 0, class F>
__device__ __forceinline__ void pw_static_for(F &&f)
{
    if constexpr (I < N) {
        f(PWInt<I>{});
        pw_static_for<N, I + 1>(f);
    }
}

struct PWArgs {
    const double *tables;
    const double *metric;  // [E][nfields][n][l][m]
    double *out;
    long long P;
    int E;
};

// Row layout of a group of NJ2 trial digits: rows are kk-major blocks (one per test
// digit kk < K of the unit) of RPK = NJ2 n2a rows rounded up to whole 8-row tiles, so
// every row tile belongs to one kk (stage B's B operand, Abar_kk, is shared by the
// tile's rows); inside a block, row r = i2 NJ2 + jj2.  off(rt) is the column offset
// (kk n1a n2a + i2 n1a, relative to the lane's row in tile 0) of row tile rt.
template <int NJ2, int K, int n1a, int n2a>
struct PWRows {
    static constexpr int RPK = ((NJ2 * n2a + 7) / 8) * 8;
    static constexpr int TPK = RPK / 8;        // row tiles per test digit
    static constexpr int NRT = K * TPK;
    static constexpr int NROWK = NJ2 * n2a;    // rows of one digit block that exist
    __host__ __device__ static constexpr int off(int rt) { return (rt / TPK) * n1a * n2a + (rt % TPK) * (8 / NJ2) * n1a; }
};

// Per-lane state of one group's stage C (see pw_group)
struct PWLane {
    int rowoff0;  // staging offset of this lane's row in row tile 0 (jj2 SEG + i2 n1a)
    int pat;      // bit x: staging pad of this lane's segment row for trial digits j1 = x mod 4
    // direct write-out (HXG_PW_WO = 1)
    double *gbase;  // &G(row 0, column I0 + i2 n1a) of this lane's row in row tile 0, minus the row start
    int Jb;         // packed row of (j1 = 0, this lane's j2)
    int thr0;       // diagonal units: columns c < J - I0 of row J are below the diagonal (-1 << 30 otherwise)
    int kc;         // test digits of the unit (row tiles of digits kk >= kc are not written)
    // staged write-out: running column state, advanced by 8 columns per step, instead of
    // divisions per step
    int bj1, bi1;        // (j1, i1) of this lane's stage-C B-operand column ct * 8 + g8
    int sj1[2], si1[2];  // (j1, i1) of this lane's D columns ct * 8 + 2 t4 + c
    int ssl[2];          // staging slot (seq + sj1) mod NSLOT
    int ej1, ei1;        // (j1, i1) of column (ct + 1) * 8: trial digits below ej1 are complete
    // bulk write-out (lanes < NJ2): packed row of the next trial digit to leave
    int wJ, wgoff, wsl;  // its row, offset of (row, column I0) in the element, staging slot
    // copy of that digit, prepared ahead of the step's DMMAs (integer work in their shadow)
    const double *bsrc;
    double *bdst;
    int blen;
};

// Source, destination and length of lane's segment of the next trial digit to leave
// (alignment fix-ups are applied at issue time).
template <int RJSEG, int SEG, int C12a>
__device__ __forceinline__ void pw_bulk_prep(PWLane &ln, const double *sS, double *outE, int epar, int I0, int kc)
{
    const int lane = threadIdx.x & 31;
    const double *slot = sS + ln.wsl * RJSEG + lane * SEG;
    const int J = ln.wJ, goff = ln.wgoff;
    const int cs = J > I0 ? J - I0 : 0;
    ln.bsrc = slot + ((epar + goff) & 1) + cs;
    ln.bdst = outE + goff + cs;
    ln.blen = kc * C12a - cs;
}

// One stage-C step: CTW column tiles starting at column tile ct, all row tiles of the
// group, then the staging stores of this lane's D fragments.
template <int S, int P, int L, int A, int B, int NJ2, int NK, int CTW, bool ASTG, int NRTA>
__device__ __forceinline__ void pw_step(const double *sT, const double *sB, double *sS, int ct, int seq,
                                        const int (&os)[NK], const int (&orr)[NK], PWLane &ln,
                                        const double (&areg)[NRTA][NK])
{
    using C = PWCfg<S, P, L>;
    constexpr int LP = C::LP, NKS = C::NKS, SEG = C::SEG, NSLOT = C::nsg(NJ2, C::RJ), RJ = C::slotrows(NJ2, C::RJ);
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n1b = C::n(B, 0);
    constexpr int NCOL = n1b * n1a;
    using R = PWRows<NJ2, C::K, n1a, n2a>;
    constexpr int NRT = R::NRT, TPK = R::TPK;
    const int lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
    // mma.sync is .aligned: the whole warp must execute it converged, and the previous
    // step ended in lane-divergent stores (independent thread scheduling does not
    // promise reconvergence there)
    __syncwarp();
    double Bp[CTW][NK];
    if constexpr (pw_direct(S)) {
#pragma unroll
        for (int w = 0; w < CTW; ++w) {
            // columns beyond NCOL read in-range table rows: their D columns are never stored
            const int col = cmin((ct + w) * 8 + g8, NCOL - 1);
            const int j1c = col / n1a, i1c = col - (col / n1a) * n1a;
            const double *ps = sT + j1c * LP, *pr = sT + i1c * LP;
#pragma unroll
            for (int ks = 0; ks < NK; ++ks) Bp[w][ks] = ps[os[ks]] * pr[orr[ks]];
        }
    } else {
        static_assert(pw_direct(S) || CTW == 1, "staged write-out runs one column tile per step");
        // columns beyond NCOL (bj1 >= n1b) read an in-range table row: never stored
        const double *ps = sT + cmin(ln.bj1, n1b - 1) * LP, *pr = sT + ln.bi1 * LP;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) Bp[0][ks] = ps[os[ks]] * pr[orr[ks]];
        ln.bi1 += 8;
        while (ln.bi1 >= n1a) { ln.bi1 -= n1a; ++ln.bj1; }
    }
    double d[CTW][NRT][2];
#pragma unroll
    for (int w = 0; w < CTW; ++w)
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) d[w][rt][0] = d[w][rt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NK; ++ks)
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) {
            double a;
            if constexpr (ASTG) a = areg[rt][ks];  // A-stationary group
            else a = sB[(rt * NKS + ks) * 32 + lane];
#pragma unroll
            for (int w = 0; w < CTW; ++w) dmma_8x8x4(d[w][rt][0], d[w][rt][1], a, Bp[w][ks]);
        }
    const bool lastv = (TPK - 1) * 8 + g8 < R::NROWK;  // this lane's row of a digit's last row tile exists
    if constexpr (pw_direct(S)) {
        constexpr int N = C::N;
#pragma unroll
        for (int w = 0; w < CTW; ++w)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int oc = (ct + w) * 8 + 2 * t4 + c;
                if (oc < NCOL) {
                    const int j1 = oc / n1a, i1 = oc - (oc / n1a) * n1a;
                    const int J = ln.Jb + j1;
                    double *dst = ln.gbase + (J * N - J * (J + 1) / 2 + i1);
                    // row-tile offsets below thr sit left of the diagonal
                    const int thr = ln.thr0 + j1 - i1;
#pragma unroll
                    for (int rt = 0; rt < NRT; ++rt)
                        if ((rt % TPK < TPK - 1 || lastv) && R::off(rt) >= thr && (C::K == 1 || rt / TPK < ln.kc)) {
                            if constexpr (HXG_PW_STCS) __stcs(dst + R::off(rt), d[w][rt][c]);
                            else dst[R::off(rt)] = d[w][rt][c];
                        }
                }
            }
    } else {
    // the slots of this step's trial digits must be free: the previous user of the
    // newest one (NSLOT digits back) committed its copies >= NSLOT - 1 - JSPAN groups ago
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(NSLOT - 1 - C::JSPAN) : "memory");
    __syncwarp();
    // store order o holds fragment column c = o ^ (t4 & 1): lanes of a quad then hit
    // columns 0, 3, 4, 7 (then 1, 2, 5, 6) -- both bank parities in one store, so the
    // even segment stride does not fold 32 lanes onto 8 of the 16 8-byte banks
    const bool sw = HXG_PW_STSWZ && (t4 & 1);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int j1 = ln.sj1[c], i1 = ln.si1[c];
        if (j1 < n1b) {
            double *base = sS + ln.ssl[c] * (RJ * SEG) + ln.rowoff0 + i1 + ((ln.pat >> (j1 & 3)) & 1);
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt)
                if ((rt % TPK < TPK - 1 || lastv) && HXG_PW_SKIP_WO < 2)
                    base[R::off(rt)] = sw ? d[0][rt][1 - c] : d[0][rt][c];
        }
        ln.si1[c] = i1 + 8;
        while (ln.si1[c] >= n1a) {
            ln.si1[c] -= n1a;
            ++ln.sj1[c];
            ln.ssl[c] = ln.ssl[c] + 1 == NSLOT ? 0 : ln.ssl[c] + 1;
        }
    }
    }
}

// One group of NJ2 trial digits j2 of a work unit: stage B into the stage-C A
// fragments, stage C (P-form) in j1 order, and the bulk write-out of every completed
// trial digit j1.
template <int S, int P, int L, int A, int B, int NJ2, int NK>
__device__ __forceinline__ void pw_group(const double *sT, double *W, double *__restrict__ outE, int epar, int j3,
                                         int I0, int kc, int j2lo, const int (&os)[NK], const int (&orr)[NK], int &seq)
{
    using C = PWCfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int LP = C::LP, N = C::N, LQ = C::LQ, LT = C::LT, NKS = C::NKS;
    constexpr int SEG = C::SEG, NSLOT = C::nsg(NJ2, C::RJ), RJ = C::slotrows(NJ2, C::RJ);
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1);
    constexpr int n1b = C::n(B, 0), n2b = C::n(B, 1);
    constexpr int sha1 = sh_of(S, A, 1), shb1 = sh_of(S, B, 1);
    constexpr int offB = C::C2::off(B);
    constexpr int C12a = n1a * n2a;
    constexpr int NCOL = n1b * n1a, NCT = (NCOL + 7) / 8;
    using R = PWRows<NJ2, C::K, n1a, n2a>;
    constexpr int NRT = R::NRT, TPK = R::TPK;
    constexpr int CTW = C::ctw(A, B);
    static_assert(NRT <= C::RTM && NJ2 <= C::RJ && 8 % NJ2 == 0, "group shape");
    const int lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
    const double *sA = W + C::W_A;
    double *sB = W + C::W_B, *sS = W + C::W_S;

    // seq = (slot of the group's first trial digit) | (NJ2 of the staging layout) << 4; a group
    // with another NJ2 re-divides the staging area, so every copy in flight must have read
    // its slot first
    if constexpr (!pw_direct(S) && HXG_PW_NSG_MAX > 0) {
        if ((seq >> 4) != NJ2) {
            bulk_wait_read();
            __syncwarp();
            seq = NJ2 << 4;
        }
    }
    const int seq0 = seq & 15;
    // this lane's rows r = rt * 8 + g8 = i2 * NJ2 + jj2 all carry jj2 = g8 % NJ2
    PWLane ln;
    {
        const int jj2 = g8 & (NJ2 - 1), i20 = g8 / NJ2;
        ln.rowoff0 = jj2 * SEG + i20 * n1a;
        // staging pad of segment (j1, jj2): parity of the packed offset of (row J, column I0),
        // J N - J (J + 1) / 2 + I0, plus the element's 8-byte phase -- a function of J mod 4
        const int Jb = offB + n1b * (j2lo + jj2 + n2b * j3);
        int pat = 0;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int J = Jb + x;
            pat |= ((epar + I0 + (J & N & 1) + ((J + 1) >> 1)) & 1) << x;
        }
        ln.pat = pat;
        ln.Jb = Jb;
        ln.gbase = outE + I0 + i20 * n1a;
        // diagonal unit (a == b, i3 == j3): I >= J <=> i1 + n1a i2 >= J - I0 = j1 + n1a (j2 - i20) ...
        ln.thr0 = Jb - I0 - i20 * n1a;
        if (!(A == B && Jb + n1b - 1 >= I0)) ln.thr0 = -(1 << 30);
        ln.kc = kc;
        // running column state (staged write-out); seq is kept reduced mod NSLOT
        ln.bj1 = g8 / n1a;
        ln.bi1 = g8 % n1a;
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // store order c <-> fragment column c ^ (t4 & 1)
            const int col = 2 * t4 + (HXG_PW_STSWZ ? (c ^ (t4 & 1)) : c);
            ln.sj1[c] = col / n1a;
            ln.si1[c] = col % n1a;
            ln.ssl[c] = (seq0 + ln.sj1[c]) % NSLOT;
        }
        ln.ej1 = 8 / n1a;
        ln.ei1 = 8 % n1a;
        const int Jw = offB + n1b * (j2lo + lane + n2b * j3);  // lanes < NJ2 own trial digit jj2 = lane
        ln.wJ = Jw;
        ln.wgoff = Jw * N - Jw * (Jw - 1) / 2 - Jw + I0;
        ln.wsl = seq0;
    }

    // ---------------- stage B: B_h[r][l] on DMMA -> stage-C A fragments ----------------
    // A-stationary: the fragments of row tile rt pass through a one-tile buffer (D layout ->
    // A layout) into registers areg[rt][*], which stage C keeps for the whole group; the
    // stage-B B operand (Abar fragments) and this lane's trial-side 1D values are loaded
    // once per group
    constexpr bool AST = pw_astat(S) || (C::K == 1 && NRT * NK <= HXG_PW_ASTAT_PAIR);
    constexpr bool HOIST = C::K == 1 && (HXG_PW_BHOIST > 1 || (AST && HXG_PW_BHOIST));
    constexpr int NRTA = AST ? NRT : 1;
    double areg[NRTA][NK];
    if constexpr (!AST) areg[0][0] = 0.0;
    constexpr int NGH = HOIST ? pp.ng : 1, LTH = HOIST ? LT : 1, LQH = HOIST ? LQ : 1;
    double agr[NGH][LTH][LQH], tbr[NGH][LQH];
    __syncwarp();  // previous group's stage C has read sB
    if constexpr (HOIST) {
        const int j2 = j2lo + (g8 & (NJ2 - 1));
#pragma unroll
        for (int g = 0; g < pp.ng; ++g) {
            const double *Tb = sT + (pp.g_fs[g] * KT + j2 + shb1) * LP;
#pragma unroll
            for (int ks = 0; ks < LQ; ++ks) {
                tbr[g][ks] = Tb[ks * 4 + t4];
#pragma unroll
                for (int lt = 0; lt < LT; ++lt) agr[g][lt][ks] = sA[(g * LT + lt) * LQ * 32 + ks * 32 + lane];
            }
        }
    } else {
        agr[0][0][0] = tbr[0][0] = 0.0;
    }
    auto stage_b_tile = [&](int rt, double *sBt) {
        constexpr CPair pp = make_pair_plan(S, A, B);  // not captured: stays a compile-time constant
        __syncwarp();  // converged for the DMMAs after the previous tile's divergent stores
        const int kk = rt / TPK, row = (rt - kk * TPK) * 8 + g8;  // row inside digit kk's block
        const int jj2 = row & (NJ2 - 1);
        const bool rv = row < R::NROWK && kk < kc;  // missing rows / digits beyond kc: zero
        const int i2 = rv ? row / NJ2 : 0;
        const int j2 = j2lo + jj2;
#pragma unroll
        for (int h = 0; h < pp.nh; ++h) {
            double d[LT][2];
#pragma unroll
            for (int lt = 0; lt < LT; ++lt) d[lt][0] = d[lt][1] = 0.0;
#pragma unroll
            for (int g = 0; g < pp.ng; ++g) {
                if (pp.g_h[g] != h) continue;
                const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sha1) * LP;
                const double *Tb = sT + (pp.g_fs[g] * KT + j2 + shb1) * LP;
                // B operand (Abar_kk) is shared by the tile's rows: every lane loads its
                // column of the tile's digit kk, rows that do not exist included
                const double *Ag = sA + (kk * C::NG + g) * LT * LQ * 32 + lane;
#pragma unroll
                for (int ks = 0; ks < LQ; ++ks) {
                    const int m = ks * 4 + t4;
                    double av;
                    if constexpr (HOIST) av = rv ? Ta[m] * tbr[g][ks] : 0.0;
                    else av = rv ? Ta[m] * Tb[m] : 0.0;
#pragma unroll
                    for (int lt = 0; lt < LT; ++lt) {
                        if constexpr (HOIST) dmma_8x8x4(d[lt][0], d[lt][1], av, agr[g][lt][ks]);
                        else dmma_8x8x4(d[lt][0], d[lt][1], av, Ag[(lt * LQ + ks) * 32]);
                    }
                }
            }
            // D[row g8][l = 8 lt + 2 t4 + c] -> A fragment (rt, k / 4), lane g8 * 4 + k % 4
#pragma unroll
            for (int lt = 0; lt < LT; ++lt)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int l = lt * 8 + 2 * t4 + c;
                    if (l < L) {
                        const int k = h * L + l;
                        sBt[(k >> 2) * 32 + g8 * 4 + (k & 3)] = d[lt][c];
                    }
                }
            __syncwarp();
        }
    };
    if constexpr (AST) {
        // forced unrolling (areg must be indexed statically to stay in registers)
        pw_static_for<NRT>([&](auto rtc) {
            constexpr int rt = decltype(rtc)::value;
            stage_b_tile(rt, sB);
#pragma unroll
            for (int ks = 0; ks < NK; ++ks) areg[rt][ks] = sB[ks * 32 + lane];
        });
    } else {
#pragma unroll 1
        for (int rt = 0; rt < NRT; ++rt) stage_b_tile(rt, sB + rt * NKS * 32);
    }
    __syncwarp();
    // ---------------- stage C: P-form on DMMA, column tiles in j1 order ----------------
    int jdone = 0;  // trial digits j1 < jdone have been written out
    constexpr int NST = NCT / CTW;  // full steps; an odd NCT ends with one single-tile step
#pragma unroll 1
    for (int st = 0; st <= NST; ++st) {
        const int ct = st * CTW;
        int jnext;
        if constexpr (!pw_direct(S)) pw_bulk_prep<RJ * SEG, SEG, C12a>(ln, sS, outE, epar, I0, kc);
        if (st < NST) {
            pw_step<S, P, L, A, B, NJ2, NK, CTW, AST>(sT, sB, sS, ct, seq, os, orr, ln, areg);
            if constexpr (pw_direct(S)) {
                jnext = ct + CTW < NCT ? ((ct + CTW) * 8) / n1a : n1b;
            } else {
                jnext = ct + 1 < NCT ? ln.ej1 : n1b;
                ln.ei1 += 8;
                while (ln.ei1 >= n1a) { ln.ei1 -= n1a; ++ln.ej1; }
            }
        } else {
            if constexpr (NCT % CTW != 0) pw_step<S, P, L, A, B, NJ2, NK, 1, AST>(sT, sB, sS, ct, seq, os, orr, ln, areg);
            jnext = n1b;
        }
        // trial digits completed by this step: one bulk copy per segment (j1, jj2)
        if (!pw_direct(S) && jnext > jdone && !HXG_PW_SKIP_WO) {
            fence_proxy_async();
            __syncwarp();
            for (int j1 = jdone; j1 < jnext; ++j1) {
                if (j1 > jdone) pw_bulk_prep<RJ * SEG, SEG, C12a>(ln, sS, outE, epar, I0, kc);
                if (lane < NJ2) {
                    const int J = ln.wJ, goff = ln.wgoff;
                    const double *src = ln.bsrc;
                    double *dst = ln.bdst;
                    int len = ln.blen;
                    if (reinterpret_cast<size_t>(dst) & 8) {
                        __stcs(dst, *src);
                        ++dst;
                        ++src;
                        --len;
                    }
                    if (len & 1) __stcs(dst + len - 1, src[len - 1]);
                    if (len >= 2) bulk_s2g(dst, src, (len & ~1) * 8);
                    // next trial digit: row J + 1 starts N - 1 - J entries further on
                    ln.wgoff = goff + (N - 1) - J;
                    ln.wJ = J + 1;
                    ln.wsl = ln.wsl + 1 == NSLOT ? 0 : ln.wsl + 1;
                }
                bulk_commit();
            }
            __syncwarp();
            jdone = jnext;
        }
    }
    if constexpr (!pw_direct(S)) seq = ((seq0 + n1b) % NSLOT) | (HXG_PW_NSG_MAX > 0 ? NJ2 << 4 : 0);  // slot of the next group's first trial digit
}

template <int S, int P, int L, int A, int B>
__device__ __forceinline__ void pw_unit(const double *sT, double *W, const double *__restrict__ M,
                                        double *__restrict__ outE, int epar, int j3, int i3, int &seq)
{
    using C = PWCfg<S, P, L>;
    constexpr CPair pp = make_pair_plan(S, A, B);
    constexpr int LP = C::LP, L3 = C::L3, LQ = C::LQ, LT = C::LT;
    const int kc = cmin(C::K, C::n(A, 2) - i3);  // test digits i3 .. i3 + kc - 1 of this unit
    constexpr int n1a = C::n(A, 0), n2a = C::n(A, 1), n2b = C::n(B, 1);
    constexpr int sha0 = sh_of(S, A, 0), sha2 = sh_of(S, A, 2);
    constexpr int shb0 = sh_of(S, B, 0), shb2 = sh_of(S, B, 2);
    constexpr int offA = C::C2::off(A);
    constexpr int KD = pp.nh * L, NK = (KD + 3) / 4;  // stage-C k-steps of this pair
    const int lane = threadIdx.x & 31, t4 = lane & 3;
    double *sP = W + C::W_P, *sA = W + C::W_A;

    // ---------------- stage A: contract xi3 -> Abar_g (stage-B B-fragment order) ----------------
    // for the unit's kc test digits at once: the metric values of a term do not depend
    // on i3, so each is loaded once and contracted with kc 1D products
    constexpr int K = C::K;
    __syncwarp();
    for (int o = lane; o < K * pp.nt * LP; o += 32) {
        const int kk = o / (pp.nt * LP), o2 = o - kk * (pp.nt * LP);
        const int t = o2 / LP, nn = o2 - t * LP;
        int fr = 0, fs = 0;
#pragma unroll
        for (int tt = 0; tt < pp.nt; ++tt)
            if (tt == t) { fr = pp.t_fr[tt]; fs = pp.t_fs[tt]; }
        const int i3k = cmin(i3 + kk, C::n(A, 2) - 1);
        sP[o] = sT[(fr * KT + i3k + sha2) * LP + nn] * sT[(fs * KT + j3 + shb2) * LP + nn];
    }
    __syncwarp();
    constexpr int NPASS = (L * L + 31) / 32;
#pragma unroll
    for (int g = 0; g < pp.ng; ++g) {
        double acc[K][NPASS];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int q = 0; q < NPASS; ++q) acc[kk][q] = 0.0;
#pragma unroll
        for (int t = 0; t < pp.nt; ++t) {
            if (pp.t_g[t] != g) continue;
            const double *Mf = M + pp.t_field[t] * L3;
            // one pass of 32 points at a time (L values per lane in flight): keeps the
            // register count low enough for 4 warps per scheduler
#pragma unroll
            for (int q = 0; q < NPASS; ++q) {
                const int lm = cmin(lane + 32 * q, L * L - 1);
                double v[L];
#pragma unroll
                for (int nn = 0; nn < L; ++nn) v[nn] = __ldg(Mf + nn * L * L + lm);
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                    const double *pt = sP + (kk * pp.nt + t) * LP;
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int nn = 0; nn < L; nn += 2) {
                        s0 = fma(v[nn], pt[nn], s0);
                        if (nn + 1 < L) s1 = fma(v[nn + 1], pt[nn + 1], s1);
                    }
                    acc[kk][q] += pp.t_sign[t] > 0 ? (s0 + s1) : -(s0 + s1);
                }
            }
        }
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
#pragma unroll
            for (int q = 0; q < NPASS; ++q) {
                const int lm = lane + 32 * q;
                if (lm < L * L) {
                    const int l = lm / L, m = lm - l * L;
                    // B fragment of tile (lt = l / 8, ks = m / 4): lane' = (l % 8) * 4 + m % 4
                    sA[(((kk * C::NG + g) * LT + (l >> 3)) * LQ + (m >> 2)) * 32 + (l & 7) * 4 + (m & 3)] = acc[kk][q];
                }
            }
    }
    __syncwarp();

    // ---------------- per-unit stage-C B-operand offsets (k = h L + l) ----------------
    int os[NK], orr[NK];
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) {
        const int k = ks * 4 + t4;
        const bool kv = k < KD;
        const int h = kv ? k / L : 0, l = kv ? k - (k / L) * L : 0;
        int fs = 0, fr = 0;
#pragma unroll
        for (int hh = 0; hh < pp.nh; ++hh)
            if (hh == h) { fs = pp.h_fs[hh]; fr = pp.h_fr[hh]; }
        // an invalid k reads a zero pad entry (l = LP - 1 >= L)
        os[ks] = kv ? (fs * KT + shb0) * LP + l : LP - 1;
        orr[ks] = kv ? (fr * KT + sha0) * LP + l : LP - 1;
    }

    const int I0 = offA + n1a * n2a * i3;
    // trial digits j2 in groups of 8, 4, 2, 1 (largest first, at most RJ; A-stationary
    // pairs also bound the fragment registers of a group)
    constexpr int RJ = pw_astat(S) ? cmin(C::RJ, pw_rj_cap(C::K, n2a, NK)) : C::RJ;
    int j2lo = 0;
#pragma unroll 1
    while (j2lo < n2b) {
        const int rem = n2b - j2lo;
#ifdef HXG_PW_SKIP_REM  // timing experiment only (wrong results): drop the groups below RJ digits
        if (rem < RJ) break;
#endif
        if (RJ >= 8 && rem >= 8) {
            if constexpr (RJ >= 8) pw_group<S, P, L, A, B, 8>(sT, W, outE, epar, j3, I0, kc, j2lo, os, orr, seq);
            j2lo += 8;
        } else if (RJ >= 4 && rem >= 4) {
            if constexpr (RJ >= 4) pw_group<S, P, L, A, B, 4>(sT, W, outE, epar, j3, I0, kc, j2lo, os, orr, seq);
            j2lo += 4;
        } else if (RJ >= 2 && rem >= 2) {
            if constexpr (RJ >= 2) pw_group<S, P, L, A, B, 2>(sT, W, outE, epar, j3, I0, kc, j2lo, os, orr, seq);
            j2lo += 2;
        } else {
            pw_group<S, P, L, A, B, 1>(sT, W, outE, epar, j3, I0, kc, j2lo, os, orr, seq);
            j2lo += 1;
        }
    }
}

template <int S, int P, int L>
__device__ __forceinline__ void pw_run_unit(int u, const double *sT, double *W, const double *__restrict__ M,
                                            double *__restrict__ outE, int epar, int &seq)
{
    using C = PWCfg<S, P, L>;
    int rem = u, pair = -1, j3 = 0, i3 = 0;
#pragma unroll
    for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int a = b; a < C::NB; ++a) {
            if (pair < 0) {
                const int n3b = C::n(b, 2), n3a = C::n(a, 2);
                int cnt = 0;  // units of the pair: test digits i3 in blocks of K
                if (a == b)
                    for (int jj = 0; jj < n3b; ++jj) cnt += C::kcnt(n3a - jj);
                else
                    cnt = n3b * C::kcnt(n3a);
                if (rem < cnt) {
                    pair = a * 3 + b;
                    if (a == b) {  // j3 <= i3 < n3, i3 = j3 + K r
                        int jj = 0, r = rem;
                        while (r >= C::kcnt(n3a - jj)) { r -= C::kcnt(n3a - jj); ++jj; }
                        j3 = jj;
                        i3 = jj + C::K * r;
                    } else {
                        j3 = rem / C::kcnt(n3a);
                        i3 = C::K * (rem - j3 * C::kcnt(n3a));
                    }
                } else {
                    rem -= cnt;
                }
            }
        }
    if constexpr (C::NB == 1) {
        pw_unit<S, P, L, 0, 0>(sT, W, M, outE, epar, j3, i3, seq);
    } else {
        switch (pair) {
        case 0: pw_unit<S, P, L, 0, 0>(sT, W, M, outE, epar, j3, i3, seq); break;
        case 3: pw_unit<S, P, L, 1, 0>(sT, W, M, outE, epar, j3, i3, seq); break;
        case 6: pw_unit<S, P, L, 2, 0>(sT, W, M, outE, epar, j3, i3, seq); break;
        case 4: pw_unit<S, P, L, 1, 1>(sT, W, M, outE, epar, j3, i3, seq); break;
        case 7: pw_unit<S, P, L, 2, 1>(sT, W, M, outE, epar, j3, i3, seq); break;
        default: pw_unit<S, P, L, 2, 2>(sT, W, M, outE, epar, j3, i3, seq); break;
        }
    }
}

// Persistent CTAs, one wave: CTA c owns the contiguous range of (element, unit)
// items [c T / G, (c + 1) T / G), T = E * NU, and its warps take the items from one
// shared-memory counter -- no barrier after the prologue, equal work per CTA
// down to one unit (small batches fill the GPU too), and the CTAs' elements
// stay few at a time (the metric of an element is read from L2 by its units).
template <int S, int P, int L>
__global__ void __launch_bounds__(PWCfg<S, P, L>::THREADS, (PWCfg<S, P, L>::MINB))
    general_pw_kernel(const __grid_constant__ PWArgs args)
{
    using C = PWCfg<S, P, L>;
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_next;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sT = smem + C::OFF_T;
    for (int idx = threadIdx.x; idx < 2 * KT * C::LP; idx += C::THREADS) {
        const int fk = idx / C::LP, l = idx - fk * C::LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    double *W = smem + C::OFF_W + warp * C::W_TOT;
    for (int idx = lane; idx < C::W_TOT; idx += 32) W[idx] = 0.0;  // zero padding of Abar / B_h
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    int seq = 0;
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
        pw_run_unit<S, P, L>((int)(item - (long long)e * C::NU), sT, W, M, outE, epar, seq);
    }
    bulk_wait_all();
}

}  // namespace hxg
