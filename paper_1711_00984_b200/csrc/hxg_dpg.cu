// hxg_dpg.cu -- the two direct consumers of the Gram kernels in the
// reference's DPG layer, batched on the device:
//
//   * the adjoint-graph Gram of the ultraweak acoustics problem
//     (/root/reference/pkg/src/hexgram/dpg.py:179-231): diagonal blocks are
//     the H1 and H(div) Grams with mass weight omega^2 + alpha (produced by
//     hxg_gram_batched), the off-diagonal block is the closed-form frequency
//     coupling S (dpg.py:155-176, graph_mixed_kernel below); the element
//     matrix is stored in real block form [[re, -im], [im, re]]
//     (dpg.py:211-219, graph_assemble_kernel);
//   * static condensation (dpg.py:348-357): A = B^T G^-1 B, rhs = B^T G^-1 l
//     through a Cholesky factor of G.  Here it is one partial Cholesky
//     elimination of the bordered matrix
//         M = [[G, B~], [B~^T, 0]],   B~ = [B | l]
//     over its first m columns: the Schur complement left in the trailing
//     (n+1) x (n+1) block is -B~^T G^-1 B~ = -[[A, rhs], [rhs^T, .]], so the
//     Cholesky factor, both triangular solves of cho_solve and the two
//     products B^T(.) are one right-looking blocked elimination
//     (condense_kernel), FP64 throughout;
//   * the sum-factorized ultraweak-acoustics stiffness B and load l
//     (dpg.py:234-302, _kernels.py:1861-1936 mixed_tens_term): 16 output
//     blocks of rectangular test x trial mixed terms, three-stage contraction
//     (xi3, xi2, xi1) per block (acoustics_block_kernel).
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/hexgram_b200.h"
#include "hxg_geom.cuh"
#include "hxg_plan.h"
#include "hxg_device.h"

using namespace hxg;

namespace {

__device__ __forceinline__ long long packed_index(long long r, long long c, long long N)
{
    if (r > c) { const long long t = r; r = c; c = t; }
    return r * N - r * (r - 1) / 2 + (c - r);
}

// ---------------------------------------------------------------------------
// adjoint-graph cross block (dpg.py:155-176):
//   S_a[(i1,i2,i3), (x1,x2,x3)] = omega (prod_d K1_d - prod_d K2_d)
//   K1_d = F01[i_d][x_d + sh_d], K2_a = F01[x_a][i_a], K2_d = K1_d (d != a),
//   sh_d = 0 on the block's own direction a, 1 elsewhere (nu_j = chi'_{j+1})
// rows: H1 flat index (i1 fastest), columns: H(div) blocks a = 0,1,2 stacked
// (dpg.py:176 np.hstack), each digit-lexicographic with x1 fastest
// (_sep3, dpg.py:146-152).  Products in the einsum's operand order.
// ---------------------------------------------------------------------------
__global__ void graph_mixed_kernel(int pr, double omega, const double *__restrict__ tab,
                                   double *__restrict__ S)
{
    const int q = pr + 1;
    const int mw = q * q * q, nb = q * pr * pr, mv = 3 * nb;
    const double *F01 = tab + TAB_F + KT * KT;
    const long long total = (long long)mw * mv;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int ih = (int)(idx / mv), iv = (int)(idx - (long long)ih * mv);
        const int a = iv / nb, x = iv - a * nb;
        const int i[3] = {ih % q, (ih / q) % q, ih / (q * q)};
        const int n0 = a == 0 ? q : pr, n1 = a == 1 ? q : pr;
        const int xd[3] = {x % n0, (x / n0) % n1, x / (n0 * n1)};
        double k1[3], k2[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d == a) {
                k1[d] = F01[i[d] * KT + xd[d]];
                k2[d] = F01[xd[d] * KT + i[d]];
            } else {
                k1[d] = k2[d] = F01[i[d] * KT + xd[d] + 1];
            }
        }
        S[idx] = omega * (k1[0] * k1[1] * k1[2] - k2[0] * k2[1] * k2[2]);
    }
}

// real block form of the adjoint-graph Gram (dpg.py:205-219):
//   G = [[re, -im], [im, re]],  re = diag(Gq, Gv),  im = [[0, S], [-S^T, 0]]
// from the packed H1 Gram gq [E][mw(mw+1)/2], the packed H(div) Gram
// gv [E][mv(mv+1)/2] and S [mw][mv] (NULL: include_mixed=False).  Writes the
// full matrices [E][2m][2m] and/or their packed upper triangles.
// one warp per output row (e, r) of the real block form: per row the source rows are
// fixed, so each output segment is a contiguous copy (packed Gram row, S row) or a
// strided gather (S column, the mirrored lower part of the full layout)
__device__ __forceinline__ void graph_row_segment(double *__restrict__ dst, int c0, int c1, int r,
                                                  int mw, int mv, const double *__restrict__ gqe,
                                                  const double *__restrict__ gve,
                                                  const double *__restrict__ S, int lane)
{
    // dst[c] for c in [c0, c1) of row r; every [c0, c1) here lies inside one quadrant
    const int m = mw + mv;
    const bool br = r >= m;
    const int R = br ? r - m : r;
    for (int c = c0 + lane; c < c1; c += 32) {
        const bool bc = c >= m;
        const int C = bc ? c - m : c;
        double v = 0.0;
        if (br == bc) {
            if (R < mw && C < mw) {
                const int lo = min(R, C), hi = max(R, C);
                v = gqe[lo * mw - lo * (lo - 1) / 2 + (hi - lo)];
            } else if (R >= mw && C >= mw) {
                const int lo = min(R, C) - mw, hi = max(R, C) - mw;
                v = gve[lo * mv - lo * (lo - 1) / 2 + (hi - lo)];
            }
        } else if (S) {
            double im = 0.0;
            if (R < mw && C >= mw) im = S[R * mv + (C - mw)];
            else if (R >= mw && C < mw) im = -S[C * mv + (R - mw)];
            v = br ? im : -im;
        }
        dst[c] = v;
    }
}

// Packed upper row r of the real block form as at most four uniform segments (a tail of a
// packed Gram row, a row or a column of S, zeros): tight copy loops instead of a branch
// tree and two integer products per entry (graph_row_segment: 55 % of the warp samples on
// the loads' scoreboard, 30 % of HBM).
__device__ __forceinline__ void graph_row_packed(double *__restrict__ dst, int r, int mw, int mv,
                                                 const double *__restrict__ gqe, const double *__restrict__ gve,
                                                 const double *__restrict__ S, int lane)
{
    // dst[c] is the entry of column c (the row pointer is already shifted by -r)
    const int m = mw + mv, M2 = 2 * m;
    const bool bottom = r >= m;
    const int R = bottom ? r - m : r;
    const int cbase = bottom ? m : 0;  // first column of the row's re quadrant
    double *d = dst;
    if (R < mw) {
        const double *src = gqe + ((long long)R * mw - (long long)R * (R - 1) / 2) - R;  // src[C], C >= R
        for (int C = R + lane; C < mw; C += 32) __stcs(d + cbase + C, src[C]);
        for (int C = mw + lane; C < m; C += 32) __stcs(d + cbase + C, 0.0);
        if (!bottom) {
            for (int C = lane; C < mw; C += 32) __stcs(d + m + C, 0.0);
            const double *sr = S ? S + (long long)R * mv : nullptr;
            for (int C = lane; C < mv; C += 32) __stcs(d + m + mw + C, sr ? -sr[C] : 0.0);
        }
    } else {
        const int lo = R - mw;
        const double *src = gve + ((long long)lo * mv - (long long)lo * (lo - 1) / 2) - lo;  // src[Cv], Cv >= lo
        for (int Cv = lo + lane; Cv < mv; Cv += 32) __stcs(d + cbase + mw + Cv, src[Cv]);
        if (!bottom) {
            for (int C = lane; C < mw; C += 32) __stcs(d + m + C, S ? S[(long long)C * mv + lo] : 0.0);
            for (int C = mw + lane; C < m; C += 32) __stcs(d + m + C, 0.0);
        }
    }
    (void)M2;
}

__global__ void graph_assemble_kernel(int mw, int mv, int E, const double *__restrict__ gq,
                                      const double *__restrict__ gv, const double *__restrict__ S,
                                      double *__restrict__ full, double *__restrict__ packed)
{
    const int M2 = 2 * (mw + mv);
    const long long NN = (long long)M2 * M2, P = (long long)M2 * (M2 + 1) / 2;
    const long long Pq = (long long)mw * (mw + 1) / 2, Pv = (long long)mv * (mv + 1) / 2;
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
         row < (long long)E * M2; row += nw) {
        const long long e = row / M2;
        const int r = (int)(row - e * M2);
        const double *gqe = gq + e * Pq, *gve = gv + e * Pv;
        if (full) {
            double *dst = full + e * NN + (long long)r * M2;
            graph_row_segment(dst, 0, M2, r, mw, mv, gqe, gve, S, lane);
        }
        if (packed) {
            double *dst = packed + e * P + (long long)r * M2 - (long long)r * (r - 1) / 2 - r;
            graph_row_packed(dst, r, mw, mv, gqe, gve, S, lane);
        }
    }
}

// ---------------------------------------------------------------------------
// static condensation (dpg.py:348-357) as a partial Cholesky elimination of
// the bordered matrix M = [[G, B~], [B~^T, 0]], B~ = [B | l], size
// Mt = m + n + 1.  Working copy: dense row-major lower triangle per element
// in the workspace (rows i >= j only).
// ---------------------------------------------------------------------------
#ifndef HXG_CD_WARPS
#define HXG_CD_WARPS 8
#endif
constexpr int CD_WARPS = HXG_CD_WARPS;
constexpr int CD_THREADS = 32 * CD_WARPS;
constexpr int CD_NB = 32;            // panel width
constexpr int CD_TT = 8 * CD_WARPS;  // trailing-update tile (rows of the panel solve: 8 per warp)
constexpr int CD_NBC = CD_TT / 16;   // 8-column DMMA tiles per warp in the trailing update

__global__ void condense_init_kernel(int m, int n, int Ec, const double *__restrict__ G,
                                     const double *__restrict__ B, const double *__restrict__ l,
                                     double *__restrict__ W)
{
    const int Mt = m + n + 1;
    const long long MM = (long long)Mt * Mt, Pg = (long long)m * (m + 1) / 2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)Ec * MM;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long e = idx / MM, rc = idx - e * MM;
        const int i = (int)(rc / Mt), j = (int)(rc - (long long)i * Mt);
        if (j > i) continue;
        double v = 0.0;
        if (i < m) {
            v = G[e * Pg + packed_index(j, i, m)];
        } else if (j < m) {
            const int r = i - m;  // border row: column r of B~
            v = r < n ? B[(e * m + j) * n + r] : (l ? l[e * m + j] : 0.0);
        }
        W[idx] = v;
    }
}

__device__ __forceinline__ void cd_dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

constexpr int CD_PS = CD_NB + 4;  // panel row stride (doubles): 8-byte fragment loads hit 16 distinct banks

// One CTA (CD_WARPS warps) per element.  Per panel of CD_NB columns:
//   (a) warp 0 factors the diagonal block L_D (unblocked, shared memory) and forms
//       L_D^-1 (one column per lane);
//   (b) per 64-row tile ti of the rows below: X = P L_D^-T as a DMMA product with the
//       explicit inverse (8 warps, in place in shared memory), written back;
//   (c) trailing update of the lower triangle W[i][j] -= sum_t X[i][t] X[j][t] for the
//       64 x 64 tiles (ti, tj <= ti), DMMA 8x8x4 with 2 x 4 accumulator tiles per warp.
__global__ void __launch_bounds__(CD_THREADS) condense_kernel(int m, int n, double *__restrict__ Wall,
                                                              int *__restrict__ status, int e0)
{
    const int Mt = m + n + 1;
    double *__restrict__ W = Wall + (long long)blockIdx.x * Mt * Mt;
    // sPi: panel rows of tile ti, [row][t]; sPj: of tile tj; sD (L_D, lower) lives in the
    // sPj space while the diagonal block is factored; sDi = L_D^-1, zero padded to CD_NB
    __shared__ __align__(16) double s_raw[2 * CD_TT * CD_PS + CD_NB * CD_PS];
    double(*sPi)[CD_PS] = reinterpret_cast<double(*)[CD_PS]>(s_raw);
    double(*sPj)[CD_PS] = reinterpret_cast<double(*)[CD_PS]>(s_raw + CD_TT * CD_PS);
    double(*sD)[CD_PS] = reinterpret_cast<double(*)[CD_PS]>(s_raw + CD_TT * CD_PS);
    double(*sDi)[CD_PS] = reinterpret_cast<double(*)[CD_PS]>(s_raw + 2 * CD_TT * CD_PS);
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    if (tid == 0) s_bad = 0;
    for (int k0 = 0; k0 < m; k0 += CD_NB) {
        const int kb = min(CD_NB, m - k0);
        // (a) diagonal block
        for (int idx = tid; idx < CD_NB * CD_NB; idx += CD_THREADS) {
            const int i = idx / CD_NB, j = idx - i * CD_NB;
            sD[i][j] = (i < kb && j <= i) ? W[(long long)(k0 + i) * Mt + k0 + j] : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
            for (int j = 0; j < kb; ++j) {
                const double d = sD[j][j];
                if (!(d > 0.0) && lane == 0) s_bad = 1;
                const double ljj = sqrt(fmax(d, 1e-300));
                __syncwarp();
                if (lane == 0) sD[j][j] = ljj;
                for (int i = j + 1 + lane; i < kb; i += 32) sD[i][j] /= ljj;
                __syncwarp();
                for (int i = j + 1 + lane; i < kb; i += 32) {
                    const double lij = sD[i][j];
                    for (int k = j + 1; k <= i; ++k) sD[i][k] = fma(-lij, sD[k][j], sD[i][k]);
                }
                __syncwarp();
            }
            // column `lane` of L_D^-1 by forward substitution
            const int j = lane;
            for (int i = 0; i < CD_NB; ++i) {
                double x = 0.0;
                if (i < kb && j < kb && i >= j) {
                    if (i == j) {
                        x = 1.0 / sD[j][j];
                    } else {
                        double sum = 0.0;
                        for (int t = j; t < i; ++t) sum = fma(sD[i][t], sDi[t][j], sum);
                        x = -sum / sD[i][i];
                    }
                }
                sDi[i][j] = x;
            }
        }
        __syncthreads();
        for (int idx = tid; idx < kb * kb; idx += CD_THREADS) {
            const int i = idx / kb, j = idx - i * kb;
            if (j <= i) W[(long long)(k0 + i) * Mt + k0 + j] = sD[i][j];
        }
        __syncthreads();  // sD (aliasing sPj) is dead from here on
        const int r0 = k0 + kb;
        const int R = Mt - r0;
        const int nt = (R + CD_TT - 1) / CD_TT;
        for (int ti = 0; ti < nt; ++ti) {
            const int ib = r0 + ti * CD_TT;
            for (int idx = tid; idx < CD_TT * CD_NB; idx += CD_THREADS) {
                const int rr = idx / CD_NB, t = idx - rr * CD_NB;
                sPi[rr][t] = (t < kb && ib + rr < Mt) ? W[(long long)(ib + rr) * Mt + k0 + t] : 0.0;
            }
            __syncthreads();
            // (b) X = P L_D^-T: warp w owns rows 8w..8w+7 of the tile (in place)
            {
                double acc[4][2];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < CD_NB / 4; ++ks) {
                    const int t = 4 * ks + t4;
                    const double a = sPi[8 * warp + g8][t];
#pragma unroll
                    for (int q = 0; q < 4; ++q) cd_dmma(acc[q][0], acc[q][1], a, sDi[8 * q + g8][t]);
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sPi[8 * warp + g8][8 * q + 2 * t4] = acc[q][0];
                    sPi[8 * warp + g8][8 * q + 2 * t4 + 1] = acc[q][1];
                }
            }
            __syncthreads();
            for (int idx = tid; idx < CD_TT * CD_NB; idx += CD_THREADS) {
                const int rr = idx / CD_NB, t = idx - rr * CD_NB;
                if (t < kb && ib + rr < Mt) W[(long long)(ib + rr) * Mt + k0 + t] = sPi[rr][t];
            }
            // (c) trailing update, warp w: rows 16 (w >> 1) .. +16, columns (CD_TT / 2) (w & 1) .. + CD_TT / 2
            const int rb = warp >> 1, cb = warp & 1;
            for (int tj = 0; tj <= ti; ++tj) {
                const int jb = r0 + tj * CD_TT;
                if (tj < ti) {
                    for (int idx = tid; idx < CD_TT * CD_NB; idx += CD_THREADS) {
                        const int rr = idx / CD_NB, t = idx - rr * CD_NB;
                        sPj[rr][t] = (t < kb && jb + rr < Mt) ? W[(long long)(jb + rr) * Mt + k0 + t] : 0.0;
                    }
                }
                __syncthreads();
                double(*Pj)[CD_PS] = tj < ti ? sPj : sPi;
                // skip warp tiles entirely above the diagonal of a diagonal tile
                const bool live = !(tj == ti && (CD_TT / 2) * cb > 16 * rb + 15);
                if (live) {
                    double acc[2][CD_NBC][2];
#pragma unroll
                    for (int a = 0; a < 2; ++a)
#pragma unroll
                        for (int b = 0; b < CD_NBC; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < CD_NB / 4; ++ks) {
                        const int t = 4 * ks + t4;
                        double av[2], bv[CD_NBC];
#pragma unroll
                        for (int a = 0; a < 2; ++a) av[a] = sPi[16 * rb + 8 * a + g8][t];
#pragma unroll
                        for (int b = 0; b < CD_NBC; ++b) bv[b] = Pj[(CD_TT / 2) * cb + 8 * b + g8][t];
#pragma unroll
                        for (int a = 0; a < 2; ++a)
#pragma unroll
                            for (int b = 0; b < CD_NBC; ++b) cd_dmma(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
                    }
#pragma unroll
                    for (int a = 0; a < 2; ++a) {
                        const int i = ib + 16 * rb + 8 * a + g8;
                        if (i >= Mt) continue;
                        double *Wi = W + (long long)i * Mt;
#pragma unroll
                        for (int b = 0; b < CD_NBC; ++b) {
                            const int j = jb + (CD_TT / 2) * cb + 8 * b + 2 * t4;
                            if (j <= i) Wi[j] -= acc[a][b][0];
                            if (j + 1 <= i) Wi[j + 1] -= acc[a][b][1];
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    __syncthreads();
    if (tid == 0 && s_bad && status) atomicOr(status + e0 + blockIdx.x, 4);
}

// A = -(Schur block)[0:n, 0:n] (mirrored), rhs = -(Schur block)[n, 0:n]
__global__ void condense_final_kernel(int m, int n, int Ec, const double *__restrict__ W,
                                      double *__restrict__ A, double *__restrict__ rhs)
{
    const int Mt = m + n + 1;
    const long long MM = (long long)Mt * Mt, NN = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)Ec * NN;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long e = idx / NN, rc = idx - e * NN;
        int r = (int)(rc / n), c = (int)(rc - (long long)r * n);
        if (c > r) { const int t = r; r = c; c = t; }
        A[idx] = -W[e * MM + (long long)(m + r) * Mt + (m + c)];
    }
    if (rhs) {
        for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)Ec * n;
             idx += (long long)gridDim.x * blockDim.x) {
            const long long e = idx / n;
            const int r = (int)(idx - e * n);
            rhs[idx] = -W[e * MM + (long long)(m + n) * Mt + (m + r)];
        }
    }
}

// ---------------------------------------------------------------------------
// ultraweak acoustics stiffness (dpg.py:234-277 _acoustics_b_tensorized) and load
// (dpg.py:280-302 _acoustics_load)
// ---------------------------------------------------------------------------
// per-point geometry fields [E][AC_NF][L^3], point (l, m, n) -> (l L + m) L + n:
//   0: 1, 1: 1/det, 2 + 3c + a: J[c][a]/det, 11 + 3d + c: Jinv[d][c]
// (the g of mixed_tens_term, _kernels.py:1899-1907)
constexpr int AC_NF = 20;

__global__ void acoustics_geom_kernel(int L, int E, const int *__restrict__ kind,
                                      const double *__restrict__ params, const double *__restrict__ tab,
                                      double *__restrict__ F, int *__restrict__ status)
{
    const int L3 = L * L * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)E * L3;
         idx += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(idx / L3), pt = (int)(idx - (long long)e * L3);
        const int l = pt / (L * L), m = (pt / L) % L, n = pt % L;
        double J[3][3];
        dev_jacobian(kind[e], params + 24LL * e, tab[TAB_NODES + l], tab[TAB_NODES + m], tab[TAB_NODES + n], J);
        const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
        const double inv = 1.0 / det;
        double Ji[3][3];
        Ji[0][0] = c00 * inv;
        Ji[1][0] = c01 * inv;
        Ji[2][0] = c02 * inv;
        Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
        Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
        Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
        Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
        Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
        Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
        double *f = F + (long long)e * AC_NF * L3 + pt;
        f[0] = 1.0;
        f[(long long)1 * L3] = 1.0 / det;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                f[(long long)(2 + 3 * c + a) * L3] = J[c][a] / det;
                f[(long long)(11 + 3 * c + a) * L3] = Ji[c][a];
            }
        if (!(det > 0.0) && status) atomicOr(status + e, 1);
    }
}

struct AcTerm {
    int su[3], sh[3], field;
    double scale;
};
struct AcBlock {
    int nterm, re;  // re: 1 -> Bre, 0 -> Bim
    int row_off, col_blk, a;  // a: H(div) component of the test rows (-1: H1 rows)
    AcTerm t[3];
};

// block b of the 16 (dpg.py:240-276, in its order); omega folded into scale
__device__ AcBlock ac_block(int b, int pr, double omega)
{
    AcBlock B{};
    const int q = pr + 1, mw = q * q * q, nb = q * pr * pr;
    if (b == 0) {  // (i omega p, q): Bim[:mw, :ny] += omega T(0,0,0; g = 1)
        B.nterm = 1; B.re = 0; B.row_off = 0; B.col_blk = 0; B.a = -1;
        B.t[0] = AcTerm{{0, 0, 0}, {0, 0, 0}, 0, omega};
    } else if (b <= 3) {  // -(u, grad q): Bre[:mw, ny(1+c)] -= sum_d T(e_d, 0; Jinv[d][c])
        const int c = b - 1;
        B.nterm = 3; B.re = 1; B.row_off = 0; B.col_blk = 1 + c; B.a = -1;
        for (int d = 0; d < 3; ++d)
            B.t[d] = AcTerm{{d == 0, d == 1, d == 2}, {0, 0, 0}, 11 + 3 * d + c, -1.0};
    } else if (b <= 6) {  // -(p, div v): Bre[off_a, :ny] -= T(1,1,1; sh_a; 1/det)
        const int a = b - 4;
        B.nterm = 1; B.re = 1; B.row_off = mw + a * nb; B.col_blk = 0; B.a = a;
        B.t[0] = AcTerm{{1, 1, 1}, {a != 0, a != 1, a != 2}, 1, -1.0};
    } else {  // (i omega u, v): Bim[off_a, ny(1+c)] += omega T(su_a, sh_a; J[c][a]/det)
        const int a = (b - 7) / 3, c = (b - 7) % 3;
        B.nterm = 1; B.re = 0; B.row_off = mw + a * nb; B.col_blk = 1 + c; B.a = a;
        B.t[0] = AcTerm{{a != 0, a != 1, a != 2}, {a != 0, a != 1, a != 2}, 2 + 3 * c + a, omega};
    }
    return B;
}

// One CTA per (block, element).  Per term: stage A (xi3) sA[l][m][i3][k3], stage B
// (xi2) sBt[l][i2][k2][i3][k3], stage C (xi1) accumulated into the block's entries in
// shared memory (sOut).  The finished block is written once to each requested output:
// its Bre or Bim part, zeros to the other part (the reference never writes those
// blocks), and the four positions of the real block form B2 = [[Bre, -Bim], [Bim, Bre]].
// Slab loop of acoustics_block_kernel.  QC (= p_r + 1 = L), N2C (= n2) and CC (= the slab's
// test digits i3, the whole extent n3) are compile-time when > 0: the index arithmetic of
// stages A and B (divisions by c p0, n2 p0 c p0, ...) then folds to constants -- with
// runtime divisors the kernel spent 60 % of its instructions on integer arithmetic
// (profiles/prof_dpg_acoustics_r01_summary.txt: IMAD 24 %, ISETP 11 %, DFMA 2 %).
template <int P0C, int QC, int N2C, int CC>
__device__ __forceinline__ void ac_slabs(int p0_arg, int pr_arg, int L_arg, int c3_arg, int e, const AcBlock &B,
                                         const double *sU, const double *sNu, const double *sW, double *sA,
                                         double *sBt, double *sOut, const double *__restrict__ F,
                                         double *__restrict__ Bre, double *__restrict__ Bim,
                                         double *__restrict__ B2)
{
    const int p0 = P0C > 0 ? P0C : p0_arg;
    const int pr = QC > 0 ? QC - 1 : pr_arg;
    const int L = QC > 0 ? QC : L_arg;
    const int q = pr + 1, mw = q * q * q, mv = 3 * q * pr * pr, m = mw + mv;
    const int ny = p0 * p0 * p0, n = 4 * ny;
    const int L3 = L * L * L;
    const int sh0 = B.t[0].sh[0], sh1 = B.t[0].sh[1], sh2 = B.t[0].sh[2];
    const int n1 = q - sh0, n2 = N2C > 0 ? N2C : q - sh1, n3 = CC > 0 ? CC : q - sh2;
    const int c3 = CC > 0 ? CC : c3_arg;
    const double *Fe = F + (long long)e * AC_NF * L3;
    // stages A and B are separable in the test digit i3: slabs of c3 digits, no recomputation
    for (int i30 = 0; i30 < n3; i30 += c3) {
        const int c = min(c3, n3 - i30);
        const int nts = n1 * n2 * c;  // rows of this slab
        for (int t = 0; t < B.nterm; ++t) {
            const AcTerm T = B.t[t];
            const double *g = Fe + (long long)T.field * L3;
            const double *u1 = sU + (T.su[0] * (q + 1) + sh0) * L;
            const double *u2 = sU + (T.su[1] * (q + 1) + sh1) * L;
            const double *u3 = sU + (T.su[2] * (q + 1) + sh2 + i30) * L;
            __syncthreads();  // tables ready / previous stage buffers consumed
            // stage A: sum over n (xi3), _kernels.py:1908-1911
            for (int i = threadIdx.x; i < L * L * c * p0; i += blockDim.x) {
                const int lm = i / (c * p0), r = i - lm * (c * p0), i3 = r / p0, k3 = r - i3 * p0;
                double s = 0.0;
                for (int nn = 0; nn < L; ++nn)
                    s = fma(sW[nn] * g[lm * L + nn], u3[i3 * L + nn] * sNu[k3 * L + nn], s);
                sA[i] = s;
            }
            __syncthreads();
            // stage B: sum over m (xi2), _kernels.py:1912-1918
            const int nb2 = n2 * p0 * c * p0;
            for (int i = threadIdx.x; i < L * nb2; i += blockDim.x) {
                const int l = i / nb2, r = i - l * nb2;
                const int i2 = r / (p0 * c * p0), r2 = r - i2 * (p0 * c * p0);
                const int k2 = r2 / (c * p0), r3 = r2 - k2 * (c * p0);  // r3 = i3 * p0 + k3
                double s = 0.0;
                for (int mm = 0; mm < L; ++mm)
                    s = fma(u2[i2 * L + mm] * sNu[k2 * L + mm] * sW[mm], sA[(l * L + mm) * c * p0 + r3], s);
                sBt[i] = s;
            }
            __syncthreads();
            // stage C: sum over l (xi1), _kernels.py:1919-1930.  A thread owns trial column
            // k (and k + kt, ...) for the rows i = rg, rg + nrg, ... of the slab: the trial
            // factors nu_k1(l) w_l sit in registers, the row digits advance incrementally
            {
                const int kt = ny < (int)blockDim.x ? ny : (int)blockDim.x;
                const int nrg = blockDim.x / kt;
                const int rg = threadIdx.x / kt, kl = threadIdx.x - rg * kt;
                if (rg < nrg) {
                    for (int k = kl; k < ny; k += kt) {
                        const int k1 = k % p0, k2 = (k / p0) % p0, k3 = k / (p0 * p0);
                        double nuw[LT];
#pragma unroll
                        for (int l = 0; l < LT; ++l) nuw[l] = l < L ? sNu[k1 * L + l] * sW[l] : 0.0;
                        const int rk = k2 * c * p0 + k3;  // r = i2 (p0 c p0) + k2 (c p0) + i3 p0 + k3
                        int i1 = rg % n1, i2 = (rg / n1) % n2, i3 = rg / (n1 * n2);
                        for (int i = rg; i < nts; i += nrg) {
                            const double *u = u1 + i1 * L;
                            const double *bt = sBt + i2 * (p0 * c * p0) + rk + i3 * p0;
                            double s = 0.0;
#pragma unroll
                            for (int l = 0; l < LT; ++l)
                                if (l < L) s = fma(u[l] * nuw[l], bt[l * nb2], s);
                            double &o = sOut[i * ny + k];  // entry owned by this thread
                            o = (t == 0 ? 0.0 : o) + T.scale * s;
                            i1 += nrg;
                            while (i1 >= n1) {
                                i1 -= n1;
                                if (++i2 == n2) { i2 = 0; ++i3; }
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        const int row0 = B.row_off + n1 * n2 * i30;
        for (int idx = threadIdx.x; idx < nts * ny; idx += blockDim.x) {
            const int i = idx / ny, k = idx - i * ny;
            const double v = sOut[idx];
            const double re = B.re ? v : 0.0, im = B.re ? 0.0 : v;
            const long long row = row0 + i, col = (long long)B.col_blk * ny + k;
            if (Bre) {
                Bre[((long long)e * m + row) * n + col] = re;
                Bim[((long long)e * m + row) * n + col] = im;
            }
            if (B2) {
                double *b2 = B2 + (long long)e * 4 * m * n;
                __stcs(b2 + row * 2 * n + col, re);
                __stcs(b2 + row * 2 * n + n + col, -im);
                __stcs(b2 + (m + row) * 2 * n + col, im);
                __stcs(b2 + (m + row) * 2 * n + n + col, re);
            }
        }
    }
}

template <int P0C, int DP>  // trial order and p_r - p0 as compile-time constants (0: runtime)
__global__ void __launch_bounds__(256) acoustics_block_kernel(int p0_arg, int pr, int L, double omega, int c3,
                                                             const double *__restrict__ tab,
                                                             const double *__restrict__ F,
                                                             double *__restrict__ Bre,
                                                             double *__restrict__ Bim,
                                                             double *__restrict__ B2)
{
    const int p0 = P0C > 0 ? P0C : p0_arg;
    extern __shared__ double sm[];
    const int b = blockIdx.x % 16, e = blockIdx.x / 16;  // 1D grid: E may exceed 65535
    const AcBlock B = ac_block(b, pr, omega);
    const int q = pr + 1, mw = q * q * q, mv = 3 * q * pr * pr, m = mw + mv;
    const int ny = p0 * p0 * p0, n = 4 * ny;
    const int L3 = L * L * L;
    const int sh0 = B.t[0].sh[0], sh1 = B.t[0].sh[1], sh2 = B.t[0].sh[2];  // shared by a block's terms
    const int n1 = q - sh0, n2 = q - sh1, n3 = q - sh2;
    // shared: 1D tables u[f][k][l] (f: chi, chi'), nu[k][l], w[l]; stage buffers for c3 digits i3
    double *sU = sm;                         // [2][q + 1][L]
    double *sNu = sU + 2 * (q + 1) * L;      // [p0][L]
    double *sW = sNu + p0 * L;               // [L]
    double *sA = sW + L;                     // [L][L][c3][p0]
    double *sBt = sA + L * L * c3 * p0;      // [L][n2][p0][c3][p0]
    double *sOut = sBt + L * n2 * p0 * c3 * p0;  // [n1 n2 c3][ny]
    for (int i = threadIdx.x; i < 2 * (q + 1) * L; i += blockDim.x) {
        const int f = i / ((q + 1) * L), r = i - f * (q + 1) * L, k = r / L, l = r - k * L;
        sU[i] = tab[TAB_T + (f * KT + k) * LT + l];
    }
    for (int i = threadIdx.x; i < p0 * L; i += blockDim.x) {
        const int k = i / L, l = i - k * L;
        sNu[i] = tab[TAB_T + (1 * KT + k + 1) * LT + l];  // nu_k = chi'_{k+1}
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) sW[i] = tab[TAB_WTS + i];
    if constexpr (P0C > 0 && DP > 0) {
        constexpr int Q = P0C + DP + 1;
        if (pr == Q - 1 && L == Q && c3 == Q) {  // default rule, whole-extent slabs
            if (sh1 == 0 && sh2 == 0) ac_slabs<P0C, Q, Q, Q>(p0, pr, L, c3, e, B, sU, sNu, sW, sA, sBt, sOut, F, Bre, Bim, B2);
            else if (sh1 == 0) ac_slabs<P0C, Q, Q, Q - 1>(p0, pr, L, c3, e, B, sU, sNu, sW, sA, sBt, sOut, F, Bre, Bim, B2);
            else if (sh2 == 0) ac_slabs<P0C, Q, Q - 1, Q>(p0, pr, L, c3, e, B, sU, sNu, sW, sA, sBt, sOut, F, Bre, Bim, B2);
            else ac_slabs<P0C, Q, Q - 1, Q - 1>(p0, pr, L, c3, e, B, sU, sNu, sW, sA, sBt, sOut, F, Bre, Bim, B2);
            return;
        }
    }
    ac_slabs<P0C, 0, 0, 0>(p0, pr, L, c3, e, B, sU, sNu, sW, sA, sBt, sOut, F, Bre, Bim, B2);
}

// dpg.py:285-302: real part of the load over the stacked test space,
// lre[e][:mw] (pressure pairing) or lre[e][mw:] (velocity pairing), other part 0.
// fgrid [E][L^3]: the source sampled at the tensor nodes (point (l, m, n)).
__global__ void acoustics_load_kernel(int pr, int L, int E, int pairing, const double *__restrict__ tab,
                                      const double *__restrict__ F, const double *__restrict__ fgrid,
                                      double *__restrict__ lre)
{
    const int q = pr + 1, mw = q * q * q, nb = q * pr * pr, m = mw + 3 * nb;
    const int L3 = L * L * L;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)E * m;
         idx += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(idx / m), i = (int)(idx - (long long)e * m);
        const double *Fe = F + (long long)e * AC_NF * L3;
        const double *fg = fgrid + (long long)e * L3;
        double s = 0.0;
        if (pairing == 1 && i < mw) {  // (f, q): w det f phi_i
            const int i1 = i % q, i2 = (i / q) % q, i3 = i / (q * q);
            for (int pt = 0; pt < L3; ++pt) {
                const int l = pt / (L * L), mm = (pt / L) % L, nn = pt % L;
                const double w = tab[TAB_WTS + l] * tab[TAB_WTS + mm] * tab[TAB_WTS + nn];
                const double phi = tab[TAB_T + i1 * LT + l] * tab[TAB_T + i2 * LT + mm] * tab[TAB_T + i3 * LT + nn];
                s += phi * (w * (1.0 / Fe[(long long)L3 + pt]) * fg[pt]);
            }
        } else if (pairing == 0 && i >= mw) {  // (f 1, J v_hat): w f sum_r J[r][a] v_a
            const int a = (i - mw) / nb, x = (i - mw) - a * nb;
            const int na0 = a == 0 ? q : pr, na1 = a == 1 ? q : pr;
            const int xd[3] = {x % na0, (x / na0) % na1, x / (na0 * na1)};
            for (int pt = 0; pt < L3; ++pt) {
                const int p3[3] = {pt / (L * L), (pt / L) % L, pt % L};
                const double w = tab[TAB_WTS + p3[0]] * tab[TAB_WTS + p3[1]] * tab[TAB_WTS + p3[2]];
                double v = 1.0;
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    v *= d == a ? tab[TAB_T + xd[d] * LT + p3[d]] : tab[TAB_T + (KT + xd[d] + 1) * LT + p3[d]];
                const double det = 1.0 / Fe[(long long)L3 + pt];
                double jr = 0.0;
#pragma unroll
                for (int c = 0; c < 3; ++c) jr += Fe[(long long)(2 + 3 * c + a) * L3 + pt] * det;
                s += (w * fg[pt]) * jr * v;
            }
        }
        lre[(long long)e * 2 * m + i] = s;
        lre[(long long)e * 2 * m + m + i] = 0.0;
    }
}

size_t ac_smem_bytes(int p0, int pr, int L, int c3)
{
    const int q = pr + 1;
    return sizeof(double) * ((size_t)2 * (q + 1) * L + (size_t)p0 * L + L + (size_t)L * L * c3 * p0 +
                             (size_t)L * q * p0 * c3 * p0 + (size_t)q * q * c3 * p0 * p0 * p0);
}

int grid_for(long long work, int threads)
{
    return (int)std::max<long long>(1, std::min<long long>((work + threads - 1) / threads, (long long)sm_count() * 16));
}

}  // namespace

extern "C" {

int hxg_graph_mixed(int pr, double omega, const double *tables, double *S, void *stream)
{
    if (pr < 1 || pr + 1 >= KT) return HXG_ERR_ORDER;
    if (!tables || !S) return HXG_ERR_ARG;
    const long long q = pr + 1, total = q * q * q * 3 * q * pr * pr;
    graph_mixed_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(pr, omega, tables, S);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

int hxg_graph_assemble(int pr, int E, const double *g_h1, const double *g_hdiv, const double *S,
                       double *full, double *packed, void *stream)
{
    if (pr < 1 || pr > HXG_MAX_ORDER) return HXG_ERR_ORDER;
    if (E < 0 || !g_h1 || !g_hdiv || (!full && !packed)) return HXG_ERR_ARG;
    if (E == 0) return HXG_OK;
    const int q = pr + 1, mw = q * q * q, mv = 3 * q * pr * pr;
    const long long M2 = 2LL * (mw + mv);
    graph_assemble_kernel<<<grid_for((long long)E * M2 * 32, 256), 256, 0, (cudaStream_t)stream>>>(
        mw, mv, E, g_h1, g_hdiv, S, full, packed);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

size_t hxg_condense_workspace_size(int m, int n, int E)
{
    if (m < 1 || n < 1 || E < 1) return 0;
    const size_t per = (size_t)(m + n + 1) * (m + n + 1) * sizeof(double);
    const size_t target = (size_t)512 << 20;  // chunk the batch to <= 512 MB of working copies
    const size_t cap = std::max<size_t>(1, target / per);
    return std::min<size_t>((size_t)E, cap) * per;
}

int hxg_condense_batched(int m, int n, int E, const double *G, const double *B, const double *l,
                         double *A, double *rhs, int *status, void *workspace, size_t ws_bytes,
                         void *stream)
{
    if (m < 1 || n < 1 || E < 0) return HXG_ERR_ARG;
    if (E == 0) return HXG_OK;
    if (!G || !B || !A) return HXG_ERR_ARG;
    const size_t per = (size_t)(m + n + 1) * (m + n + 1) * sizeof(double);
    if (!workspace || ws_bytes < per) return HXG_ERR_WORKSPACE;
    const int chunk = (int)std::min<size_t>((size_t)E, ws_bytes / per);
    cudaStream_t st = (cudaStream_t)stream;
    double *W = (double *)workspace;
    if (status && cudaMemsetAsync(status, 0, sizeof(int) * (size_t)E, st) != cudaSuccess) return HXG_ERR_CUDA;
    const long long Pg = (long long)m * (m + 1) / 2;
    for (int e0 = 0; e0 < E; e0 += chunk) {
        const int Ec = std::min(chunk, E - e0);
        const long long Mt = m + n + 1;
        condense_init_kernel<<<grid_for((long long)Ec * Mt * Mt, 256), 256, 0, st>>>(
            m, n, Ec, G + e0 * Pg, B + (long long)e0 * m * n, l ? l + (long long)e0 * m : nullptr, W);
        condense_kernel<<<Ec, CD_THREADS, 0, st>>>(m, n, W, status, e0);
        condense_final_kernel<<<grid_for((long long)Ec * n * n, 256), 256, 0, st>>>(
            m, n, Ec, W, A + (long long)e0 * n * n, rhs ? rhs + (long long)e0 * n : nullptr);
    }
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

size_t hxg_acoustics_workspace_size(int p0, int pr, int L, int E)
{
    if (p0 < 1 || pr < 1 || L < 1 || E < 0) return 0;
    return sizeof(double) * (size_t)E * AC_NF * L * L * L;
}

int hxg_acoustics_batched(int p0, int pr, double omega, int L, int E, const int *kind,
                          const double *params, const double *tables, const double *fgrid, int pairing,
                          double *Bre, double *Bim, double *B2, double *lre, int *status,
                          void *workspace, size_t ws_bytes, void *stream)
{
    if (p0 < 1 || pr < p0 || pr + 2 > KT || L < 1 || L > LT) return HXG_ERR_ORDER;
    if (E < 0 || pairing < 0 || pairing > 1) return HXG_ERR_ARG;
    if (E == 0) return HXG_OK;
    if (!kind || !params || !tables || (!Bre != !Bim) || (!Bre && !B2) || (lre && !fgrid)) return HXG_ERR_ARG;
    if (!workspace || ws_bytes < hxg_acoustics_workspace_size(p0, pr, L, E)) return HXG_ERR_WORKSPACE;
    int c3 = pr + 1;  // i3 slab: the largest that fits the shared-memory budget
    while (c3 > 1 && ac_smem_bytes(p0, pr, L, c3) > 200 * 1024) --c3;
    const size_t smem = ac_smem_bytes(p0, pr, L, c3);
    if (smem > 227 * 1024) return HXG_ERR_ORDER;
    const int m = (pr + 1) * (pr + 1) * (pr + 1) + 3 * (pr + 1) * pr * pr;
    cudaStream_t st = (cudaStream_t)stream;
    double *F = (double *)workspace;
    if (status && cudaMemsetAsync(status, 0, sizeof(int) * (size_t)E, st) != cudaSuccess) return HXG_ERR_CUDA;
    acoustics_geom_kernel<<<grid_for((long long)E * L * L * L, 256), 256, 0, st>>>(L, E, kind, params, tables,
                                                                                  F, status);
    auto kern = acoustics_block_kernel<0, 0>;
    const int dp = pr - p0;
    switch (p0) {
#define HXG_AC_CASE(PP)                                                                   \
    case PP:                                                                              \
        kern = dp == 1 ? acoustics_block_kernel<PP, 1>                                    \
                       : (dp == 2 ? acoustics_block_kernel<PP, 2> : acoustics_block_kernel<PP, 0>); \
        break;
        HXG_AC_CASE(1) HXG_AC_CASE(2) HXG_AC_CASE(3) HXG_AC_CASE(4)
#undef HXG_AC_CASE
    case 5: kern = acoustics_block_kernel<5, 0>; break;
    case 6: kern = acoustics_block_kernel<6, 0>; break;
    default: break;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return HXG_ERR_CUDA;
    kern<<<16 * E, 256, smem, st>>>(p0, pr, L, omega, c3, tables, F, Bre, Bim, B2);
    if (lre)
        acoustics_load_kernel<<<grid_for((long long)E * m, 128), 128, 0, st>>>(pr, L, E, pairing, tables, F,
                                                                             fgrid, lre);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

}  // extern "C"
