// hxg_kernels.cuh -- sm_100a device code for the batched Gram integration.
//
//   tables_kernel   1D tables on device: Gauss-Legendre (quadrature.py:47-66),
//                   chi / chi' at the nodes (_kernels.py:29-43), closed-form
//                   F tables (poly1d.py:140-266)
//   metric_kernel   per-point Jacobian, det, inverse, D = J^-1 J^-T, C = J^T J
//                   (_kernels.py:56-136) folded with the quadrature weight and the
//                   mass coefficient into the term fields of hxg_plan.h
//   general_kernel  three-stage sum factorization (tens_*, _kernels.py:356-1150)
//                   stage A/B on DFMA in shared memory, stage C on FP64 DMMA
//                   (mma.sync m8n8k4 f64 -> DMMA.8x8x4), output staged in
//                   shared memory and streamed to HBM as contiguous row segments
//   affine_kernel   constant-Jacobian O(p^6) path (simp_*_const,
//                   _kernels.py:1169-1404): closed-form F-table products,
//                   write-bandwidth bound
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "hxg_common.cuh"
#include "hxg_geom.cuh"

namespace hxg {

constexpr int AFF_THREADS = 128;
constexpr int MAX_UNITS = 48;  // (block, digit) work units per element: 3 * 13 = 39

struct GenArgs {
    SpacePlan plan;
    int L, LP, E;            // rule points, padded stride (even), elements in this launch
    int R2, R3;              // j2 rows / i3 columns per chunk
    int N2, NG, NH;          // capacities used for shared-memory strides
    int SLD;                 // staging row stride (doubles)
    int nunits;
    int8_t unit_b[MAX_UNITS], unit_j3[MAX_UNITS];
    int off_T, off_A, off_B, off_S;  // shared-memory offsets (doubles)
    const double *tables;    // TAB_TOTAL doubles
    const double *metric;    // [E][nfields][L^3]
    double *out;             // [E][P]
    long long P;             // N(N+1)/2
};

struct AffArgs {
    SpacePlan plan;
    int E, nunits_total;     // row groups per element
    int ucount[3];           // row groups per block b: n[b][1] * n[b][2]
    int N2, N3;              // capacities for the B-sum table
    const int *kind;
    const double *params, *coef, *tables;
    double *out;
    int *status;
    long long P;
};

// ---------------------------------------------------------------------------
// 1D tables
// ---------------------------------------------------------------------------
// The 1D tables follow the reference's arithmetic operation for operation, with
// every product / sum rounded separately (no FMA contraction: numba compiles the
// reference without fast-math), so the device rule and shape tables equal the
// reference arrays to the last bit up to the cos() of the Newton start.
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }

// P_L(x), P_L'(x) (quadrature.py:37-44): p = ((2k-1) x p - (k-1) p_prev) / k,
// dp = L (x p - p_prev) / (x x - 1)
__device__ inline void dev_legendre_pl(int L, double x, double &p, double &dp)
{
    double pm = 1.0, pc = x;
    for (int k = 2; k <= L; ++k) {
        const double pn = rn_div(rn_sub(rn_mul(rn_mul((double)(2 * k - 1), x), pc), rn_mul((double)(k - 1), pm)),
                                 (double)k);
        pm = pc;
        pc = pn;
    }
    p = pc;
    dp = rn_div(rn_mul((double)L, rn_sub(rn_mul(x, pc), pm)), rn_sub(rn_mul(x, x), 1.0));
}

__device__ inline double dev_f00(int i, int j)
{
    if (i < j) { int t = i; i = j; j = t; }
    if (j >= 2) {
        if (i == j) return (1.0 / (2 * j + 1) + 1.0 / (2 * j - 3)) / (4.0 * (2 * j - 1) * (2 * j - 1));
        if (i == j + 2) return -1.0 / (4.0 * (2 * j + 3) * (2 * j - 1) * (2 * j + 1));
        return 0.0;
    }
    if (j == 1) return i == 1 ? 1.0 / 3.0 : i == 2 ? -1.0 / 12.0 : i == 3 ? -1.0 / 60.0 : 0.0;
    return i == 0 ? 1.0 / 3.0 : i == 1 ? 1.0 / 6.0 : i == 2 ? -1.0 / 12.0 : i == 3 ? 1.0 / 60.0 : 0.0;
}

__device__ inline double dev_f01(int i, int j)
{
    double sg = 1.0;
    if (j == 0) { j = 1; sg = -1.0; }  // chi_0' = -chi_1'
    double v;
    if (i == 0) v = j == 1 ? 0.5 : j == 2 ? -1.0 / 6.0 : 0.0;
    else if (i == 1) v = j == 1 ? 0.5 : j == 2 ? 1.0 / 6.0 : 0.0;
    else if (i == 2) v = j == 1 ? -1.0 / 6.0 : j == 3 ? 1.0 / 30.0 : 0.0;
    else if (j == i + 1) v = 1.0 / (2.0 * (2 * i - 1) * (2 * i + 1));
    else if (j == i - 1) v = -1.0 / (2.0 * (2 * i - 1) * (2 * i - 3));
    else v = 0.0;
    return sg * v;
}

__device__ inline double dev_f11(int i, int j)
{
    if (i < j) { int t = i; i = j; j = t; }
    if (j >= 1) return i == j ? 1.0 / (2 * i - 1) : 0.0;
    return i == 0 ? 1.0 : i == 1 ? -1.0 : 0.0;
}

__global__ void tables_kernel(int L, const double *__restrict__ user_nodes,
                              const double *__restrict__ user_wts, double *__restrict__ tab)
{
    __shared__ double s_nodes[LT];
    const int tid = threadIdx.x;
    if (tid < 32) {  // one warp: L <= LT = 16 nodes
        const bool act = tid < L;
        double node = 0.0, wt = 0.0;
        if (user_nodes) {
            if (act) {
                node = user_nodes[tid];
                wt = user_wts[tid];
            }
        } else if (L == 1) {
            if (act) {
                node = 0.5;
                wt = 1.0;
            }
        } else {
            // quadrature.py:53-65: x_k = cos(pi (k - 1/4) / (L + 1/2)), k = 1..L, all nodes
            // updated together until max |dx| < 1e-15; lane tid holds k = L - tid so the
            // mapped nodes increase with tid (nodes = 0.5 (1 + x[::-1]))
            const int k = L - tid;
            double x = act ? cos(rn_div(rn_mul(M_PI, rn_sub((double)k, 0.25)), rn_add((double)L, 0.5))) : 0.0;
            for (int it = 0; it < 100; ++it) {
                double p = 0.0, dp = 1.0;
                if (act) dev_legendre_pl(L, x, p, dp);
                const double dx = act ? rn_div(p, dp) : 0.0;
                x = rn_sub(x, dx);
                double m = fabs(dx);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                if (m < 1e-15) break;
            }
            double p = 0.0, dp = 1.0;
            if (act) dev_legendre_pl(L, x, p, dp);
            if (act) {
                const double w = rn_div(2.0, rn_mul(rn_mul(rn_sub(1.0, rn_mul(x, x)), dp), dp));
                node = rn_mul(0.5, rn_add(1.0, x));
                wt = rn_mul(0.5, w);
            }
        }
        if (tid < LT) {
            tab[TAB_NODES + tid] = node;
            tab[TAB_WTS + tid] = wt;
            s_nodes[tid] = node;
        }
    }
    __syncthreads();
    // chi_k, chi'_k at each node (_kernels.py:29-43 with p = KT - 1)
    if (tid < LT) {
        const double xi = s_nodes[tid];
        const double t = rn_sub(rn_mul(2.0, xi), 1.0);
        double *chi = tab + TAB_T, *dchi = tab + TAB_T + KT * LT;
        chi[0 * LT + tid] = rn_sub(1.0, xi);
        chi[1 * LT + tid] = xi;
        dchi[0 * LT + tid] = -1.0;
        dchi[1 * LT + tid] = 1.0;
        double pm2 = 1.0, pm1 = t;
        for (int i = 2; i < KT; ++i) {
            const double pi = rn_div(rn_sub(rn_mul(rn_mul((double)(2 * i - 1), t), pm1), rn_mul((double)(i - 1), pm2)),
                                     (double)i);
            chi[i * LT + tid] = rn_div(rn_sub(pi, pm2), rn_mul(2.0, (double)(2 * i - 1)));
            dchi[i * LT + tid] = pm1;
            pm2 = pm1;
            pm1 = pi;
        }
    }
    // F tables, stacked [F00, F01, F10 = F01^T, F11] (poly1d.py:265)
    for (int idx = tid; idx < KT * KT; idx += blockDim.x) {
        const int i = idx / KT, j = idx % KT;
        tab[TAB_F + 0 * KT * KT + idx] = dev_f00(i, j);
        tab[TAB_F + 1 * KT * KT + idx] = dev_f01(i, j);
        tab[TAB_F + 2 * KT * KT + idx] = dev_f01(j, i);
        tab[TAB_F + 3 * KT * KT + idx] = dev_f11(i, j);
    }
}

// ---------------------------------------------------------------------------
// per-point metric kernel: metric[e][field][(l L + m) L + n]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) metric_kernel(int space, int L, int E,
                                                     const int *__restrict__ kind,
                                                     const double *__restrict__ params,
                                                     const double *__restrict__ coef,
                                                     const double *__restrict__ wgrid,
                                                     const double *__restrict__ tab,
                                                     double *__restrict__ metric,
                                                     int *__restrict__ status, int nfields)
{
    const int L3 = L * L * L;
    const long long total = (long long)E * L3;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(idx / L3);
        const int pt = (int)(idx - (long long)e * L3);
        // metric layout [e][field][n][l][m]: lanes run along m (coalesced stage-A reads)
        const int n = pt / (L * L), l = (pt / L) % L, m = pt % L;
        const double *par = params + 24LL * e;
        double J[3][3], D[6], C[6], f[MAXF];
        dev_jacobian(kind[e], par, tab[TAB_NODES + l], tab[TAB_NODES + m], tab[TAB_NODES + n], J);
        const double det = dev_metrics(J, D, C);
        const double w = tab[TAB_WTS + l] * tab[TAB_WTS + m] * tab[TAB_WTS + n];
        const double c = wgrid ? wgrid[(long long)e * L3 + (l * L + m) * L + n] : (coef ? coef[e] : 1.0);
        dev_fields(space, det, D, C, w, c, f);
        double *mo = metric + (long long)e * nfields * L3 + pt;
        for (int k = 0; k < nfields; ++k) mo[(long long)k * L3] = f[k];
        if (!(det > 0.0)) atomicOr(status + e, 1);
    }
}

// ---------------------------------------------------------------------------
// general map: three-stage sum factorization
// ---------------------------------------------------------------------------

// Work unit = (element e, trial block b, trial digit j3): the rows J of the packed
// output with block b and digit j3, i.e. one contiguous range of packed rows.
// Columns are processed in chunks (test block a >= b, i3 range of R3 digits);
// rows in groups of R2 values of j2 (all j1).
template <int LMAX, int NMT>
__global__ void __launch_bounds__(GEN_THREADS, (LMAX <= 8 ? 2 : 1))
    general_kernel(const __grid_constant__ GenArgs args)
{
    extern __shared__ __align__(16) double smem[];
    const SpacePlan &P = args.plan;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int L = args.L, LP = args.LP, L3 = L * L * L;
    const int R2 = args.R2, R3 = args.R3, N2 = args.N2, NG = args.NG, NH = args.NH;
    const int SLD = args.SLD;
    const int u = blockIdx.x % args.nunits;
    const int e = blockIdx.x / args.nunits;
    const int b = args.unit_b[u], j3 = args.unit_j3[u];
    const int N = P.N;

    double *sT = smem + args.off_T;  // [2][KT][LP]
    double *sA = smem + args.off_A;  // [R3][NG][L][LP]      Abar_g(l, m) stored [m][l]
    double *sB = smem + args.off_B;  // [R2][NH][R3][N2][LP] B_h(l)
    double *sS = smem + args.off_S;  // [R2 * n1b][SLD]      output staging
    const int SJ2 = NH * R3 * N2 * LP;

    for (int idx = tid; idx < 2 * KT * LP; idx += GEN_THREADS) {
        const int fk = idx / LP, l = idx - fk * LP;
        sT[idx] = l < L ? args.tables[TAB_T + fk * LT + l] : 0.0;
    }
    const double *__restrict__ M = args.metric + (long long)e * P.nfields * L3;
    double *__restrict__ outE = args.out + (long long)e * args.P;

    const int n1b = P.n[b][0], n2b = P.n[b][1], n3b = P.n[b][2];
    (void)n3b;
    const int shb0 = P.sh[b][0], shb1 = P.sh[b][1], shb2 = P.sh[b][2];

    for (int a = b; a < P.nb; ++a) {
        const PairPlan &pp = P.pair[a][b];
        const int n1a = P.n[a][0], n2a = P.n[a][1], n3a = P.n[a][2];
        const int sha0 = P.sh[a][0], sha1 = P.sh[a][1], sha2 = P.sh[a][2];
        const int kdim = pp.nh * L;
        const int nks = (kdim + 3) >> 2;
        __syncthreads();  // sT ready / previous chunk done with sA
        // A fragments (trial side): A[j1][k] = u_{s1(h)}(j1 + sh, l), k = h L + l
        double Af[NMT][LMAX];
#pragma unroll
        for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
            for (int ks = 0; ks < LMAX; ++ks) {
                const int j1 = mt * 8 + g8, k = ks * 4 + t4;
                double v = 0.0;
                if (ks < nks && k < kdim && j1 < n1b) {
                    const int h = k / L, l = k - h * L;
                    v = sT[(pp.h_fs[h] * KT + j1 + shb0) * LP + l];
                }
                Af[mt][ks] = v;
            }
        const int i3first = (a == b) ? j3 : 0;
        for (int i3lo = i3first; i3lo < n3a; i3lo += R3) {
            const int r3 = min(R3, n3a - i3lo);
            const int ncols = n1a * n2a * r3;
            const int nct = (ncols + 7) >> 3;
            // ---------------- stage A: contract xi3 (n) ----------------
            {
                const int items = r3 * pp.ng * L * L;
                for (int it = tid; it < items; it += GEN_THREADS) {
                    int rest = it;
                    const int m = rest % L; rest /= L;
                    const int l = rest % L; rest /= L;
                    const int g = rest % pp.ng;
                    const int ii3 = rest / pp.ng;
                    const int i3 = i3lo + ii3;
                    double acc = 0.0;
                    for (int t = 0; t < pp.nt; ++t) {
                        if (pp.t_g[t] != g) continue;
                        const double *__restrict__ Mf = M + pp.t_field[t] * L3 + l * L + m;
                        const double *Ta = sT + (pp.t_fr[t] * KT + i3 + sha2) * LP;
                        const double *Tb = sT + (pp.t_fs[t] * KT + j3 + shb2) * LP;
                        double s = 0.0;
                        for (int n = 0; n < L; ++n) s += __ldg(Mf + n * L * L) * (Ta[n] * Tb[n]);
                        acc += pp.t_sign[t] > 0 ? s : -s;
                    }
                    sA[((ii3 * NG + g) * L + m) * LP + l] = acc;
                }
            }
            for (int j2lo = 0; j2lo < n2b; j2lo += R2) {
                const int r2 = min(R2, n2b - j2lo);
                __syncthreads();  // sA complete; previous stage C done with sB
                // ---------------- stage B: contract xi2 (m) ----------------
                {
                    const int items = r2 * pp.nh * r3 * n2a;
                    for (int it = tid; it < items; it += GEN_THREADS) {
                        int rest = it;
                        const int i2 = rest % n2a; rest /= n2a;
                        const int ii3 = rest % r3; rest /= r3;
                        const int h = rest % pp.nh;
                        const int jj2 = rest / pp.nh;
                        const int j2 = j2lo + jj2;
                        double acc[LMAX];
#pragma unroll
                        for (int l = 0; l < LMAX; ++l) acc[l] = 0.0;
                        for (int g = 0; g < pp.ng; ++g) {
                            if (pp.g_h[g] != h) continue;
                            const double *Ta = sT + (pp.g_fr[g] * KT + i2 + sha1) * LP;
                            const double *Tb = sT + (pp.g_fs[g] * KT + j2 + shb1) * LP;
                            const double *Ag = sA + (ii3 * NG + g) * L * LP;
                            for (int m = 0; m < L; ++m) {
                                const double v = Ta[m] * Tb[m];
                                const double2 *Am = reinterpret_cast<const double2 *>(Ag + m * LP);
#pragma unroll
                                for (int l2 = 0; l2 < LMAX / 2; ++l2) {
                                    if (2 * l2 < L) {
                                        const double2 av = Am[l2];
                                        acc[2 * l2] += av.x * v;
                                        acc[2 * l2 + 1] += av.y * v;
                                    }
                                }
                            }
                        }
                        double *dst = sB + jj2 * SJ2 + ((h * R3 + ii3) * N2 + i2) * LP;
#pragma unroll
                        for (int l = 0; l < LMAX; ++l)
                            if (l < L) dst[l] = acc[l];
                    }
                }
                __syncthreads();
                // ---------------- stage C: contract xi1 (l) on DMMA ----------------
                for (int ct = warp; ct < nct; ct += GEN_WARPS) {
                    const int c = ct * 8 + g8;
                    const bool cval = c < ncols;
                    const int i1 = c % n1a, rest = c / n1a, i2 = rest % n2a, ii3 = rest / n2a;
                    double X[LMAX];
                    int bo[LMAX];
#pragma unroll
                    for (int ks = 0; ks < LMAX; ++ks) {
                        const int k = ks * 4 + t4;
                        X[ks] = 0.0;
                        bo[ks] = 0;
                        if (ks < nks && k < kdim && cval) {
                            const int h = k / L, l = k - h * L;
                            X[ks] = sT[(pp.h_fr[h] * KT + i1 + sha0) * LP + l];
                            bo[ks] = ((h * R3 + ii3) * N2 + i2) * LP + l;
                        }
                    }
                    for (int jj2 = 0; jj2 < r2; ++jj2) {
                        __syncwarp();  // converged for mma.sync (.aligned) after divergent code
                        const double *sBj = sB + jj2 * SJ2;
                        double d[NMT][2];
#pragma unroll
                        for (int mt = 0; mt < NMT; ++mt) d[mt][0] = d[mt][1] = 0.0;
#pragma unroll
                        for (int ks = 0; ks < LMAX; ++ks) {
                            if (ks < nks) {
                                const double bv = X[ks] * sBj[bo[ks]];
#pragma unroll
                                for (int mt = 0; mt < NMT; ++mt) dmma_8x8x4(d[mt][0], d[mt][1], Af[mt][ks], bv);
                            }
                        }
#pragma unroll
                        for (int mt = 0; mt < NMT; ++mt) {
                            const int j1 = mt * 8 + g8;
                            if (j1 < n1b) {
                                double2 *dst = reinterpret_cast<double2 *>(
                                    sS + (jj2 * n1b + j1) * SLD + ct * 8 + 2 * t4);
                                *dst = make_double2(d[mt][0], d[mt][1]);
                            }
                        }
                    }
                }
                __syncthreads();
                // ---------------- write-out: contiguous packed row segments ----------------
                {
                    const int rows = r2 * n1b;
                    const long long I0 = P.off[a] + (long long)n1a * n2a * i3lo;
                    for (int row = warp; row < rows; row += GEN_WARPS) {
                        const int jj2 = row / n1b, j1 = row - jj2 * n1b;
                        const long long J = P.off[b] + j1 + (long long)n1b * (j2lo + jj2 + (long long)n2b * j3);
                        long long cs = J - I0;
                        if (cs < 0) cs = 0;
                        double *rowp = outE + J * N - J * (J - 1) / 2 - J + I0;  // &G(J, I0)
                        const double *src = sS + row * SLD;
                        for (long long cc = cs + lane; cc < ncols; cc += 32) __stcs(rowp + cc, src[cc]);
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// constant-Jacobian map: closed-form F-table products
// ---------------------------------------------------------------------------
// Work unit = (element e, trial block b, trial digits j2, j3): the n1b packed rows
// J = (j1, j2, j3, b), written in full from column J to N - 1.
__global__ void __launch_bounds__(AFF_THREADS) affine_kernel(const __grid_constant__ AffArgs args)
{
    extern __shared__ __align__(16) double smem[];
    const SpacePlan &P = args.plan;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int e = blockIdx.x / args.nunits_total;
    int u = blockIdx.x - e * args.nunits_total;
    const bool first_unit = (u == 0);
    int b = 0;
    while (u >= args.ucount[b]) { u -= args.ucount[b]; ++b; }
    const int n1b = P.n[b][0], n2b = P.n[b][1];
    const int j2 = u % n2b, j3 = u / n2b;
    const int N = P.N, N2 = args.N2, N3 = args.N3;

    double *sF = smem;                        // [4][KT][KT]
    double *sBs = smem + 4 * KT * KT;         // [3][N3][N2][MAXH]
    __shared__ double s_field[MAXF];

    for (int idx = tid; idx < 4 * KT * KT; idx += AFF_THREADS) sF[idx] = args.tables[TAB_F + idx];
    if (tid == 0) {
        double J[3][3], D[6], C[6];
        dev_jacobian(args.kind[e], args.params + 24LL * e, 0.5, 0.5, 0.5, J);
        const double det = dev_metrics(J, D, C);
        const double c = args.coef ? args.coef[e] : 1.0;
        dev_fields(P.space, det, D, C, 1.0, c, s_field);
        if (first_unit) {
            if (!(det > 0.0)) atomicOr(args.status + e, 1);
            if (args.kind[e] > 2) atomicOr(args.status + e, 2);  // gram.py:170-174
        }
    }
    __syncthreads();
    // B-sums: Bs[a][i3][i2][h] = sum_{g in h} F_g(i2, j2) sum_{t in g} sign field F_t(i3, j3)
    for (int a = b; a < P.nb; ++a) {
        const PairPlan &pp = P.pair[a][b];
        const int n2a = P.n[a][1], n3a = P.n[a][2];
        const int items = n3a * n2a;
        for (int it = tid; it < items; it += AFF_THREADS) {
            const int i2 = it % n2a, i3 = it / n2a;
            double acc[MAXH] = {0.0, 0.0, 0.0, 0.0};
            for (int g = 0; g < pp.ng; ++g) {
                double sa = 0.0;
                for (int t = 0; t < pp.nt; ++t) {
                    if (pp.t_g[t] != g) continue;
                    const double f = sF[((2 * pp.t_fr[t] + pp.t_fs[t]) * KT + i3 + P.sh[a][2]) * KT + j3 + P.sh[b][2]];
                    const double v = s_field[pp.t_field[t]] * f;
                    sa += pp.t_sign[t] > 0 ? v : -v;
                }
                const double fb = sF[((2 * pp.g_fr[g] + pp.g_fs[g]) * KT + i2 + P.sh[a][1]) * KT + j2 + P.sh[b][1]];
                const int h = pp.g_h[g];
#pragma unroll
                for (int hh = 0; hh < MAXH; ++hh)
                    if (hh == h) acc[hh] += fb * sa;
            }
            double *dst = sBs + ((a * N3 + i3) * N2 + i2) * MAXH;
#pragma unroll
            for (int hh = 0; hh < MAXH; ++hh) dst[hh] = acc[hh];
        }
    }
    __syncthreads();
    double *__restrict__ outE = args.out + (long long)e * args.P;
    for (int j1 = warp; j1 < n1b; j1 += AFF_THREADS / 32) {
        const long long J = P.off[b] + j1 + (long long)n1b * (j2 + (long long)n2b * j3);
        double *rowp = outE + J * N - J * (J - 1) / 2 - J;  // &G(J, 0)
        for (long long I = J + lane; I < N; I += 32) {
            int a = 0;
            if (P.nb > 1) a = (I >= P.off[2]) ? 2 : (I >= P.off[1] ? 1 : 0);
            const PairPlan &pp = P.pair[a][b];
            const int n1a = P.n[a][0], n2a = P.n[a][1];
            const int rem = (int)(I - P.off[a]);
            const float inv1 = 1.0f / n1a, inv2 = 1.0f / n2a;
            const int q1 = (int)((rem + 0.5f) * inv1);
            const int i1 = rem - q1 * n1a;
            const int i3 = (int)((q1 + 0.5f) * inv2);
            const int i2 = q1 - i3 * n2a;
            const double *bs = sBs + ((a * N3 + i3) * N2 + i2) * MAXH;
            double v = 0.0;
            for (int h = 0; h < pp.nh; ++h)
                v += sF[((2 * pp.h_fr[h] + pp.h_fs[h]) * KT + i1 + P.sh[a][0]) * KT + j1 + P.sh[b][0]] * bs[h];
            __stcs(rowp + I, v);
        }
    }
}

// packed upper triangle -> full symmetric matrix
// status bit 1 for kinds without an extrusion/constant-Jacobian structure on the
// simplified extrusion path (gram.py:170-174), when the general kernels serve it
__global__ void ext_kind_kernel(int E, const int *__restrict__ kind, int *__restrict__ status)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E && kind[e] > 3) atomicOr(status + e, 2);
}

__global__ void expand_kernel(int N, long long total, const double *__restrict__ packed,
                              double *__restrict__ full)
{
    const long long NN = (long long)N * N;
    const long long P = (long long)N * (N + 1) / 2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long e = idx / NN;
        const long long rc = idx - e * NN;
        long long r = rc / N, c = rc - r * N;
        if (r > c) { long long t = r; r = c; c = t; }
        full[idx] = packed[e * P + r * N - r * (r - 1) / 2 + (c - r)];
    }
}

}  // namespace hxg
