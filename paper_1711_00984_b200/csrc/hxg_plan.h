// hxg_plan.h -- space descriptors shared by the host planner and the
// sm_100a kernels.
//
// Every Gram integrand of the reference (restated by the einsum oracle at
// /root/reference/pkg/tests/test_gram.py:22-44, weighted as in
// /root/reference/pkg/src/hexgram/_kernels.py:206-348) is, for one pair of
// component blocks (a, b), a signed sum of TERMS
//
//     sign * field_k(xi) * prod_d u^{a,d}_{r_d}(i_d, xi_d) * u^{b,d}_{s_d}(j_d, xi_d)
//
// where field_k is a per-point metric scalar (c det, D_ab det, C_ab/det,
// 1/det ... times the quadrature weight) and u^{a,d}_r is one of the two 1D
// functions chi_k, chi'_k evaluated at digit i_d + shift(a, d).  Sum
// factorization contracts xi3 (stage A), xi2 (stage B) and xi1 (stage C).
// The planner groups terms that share their xi1/xi2 factor pairs so that each
// stage sums them once:
//   stage A term t -> group g = (r1, s1, r2, s2)   ("Abar_g")
//   stage B group g -> group h = (r1, s1)          ("B_h")
//   stage C: G[I, J] = sum_h sum_l u_{r1}(i1, l) u_{s1}(j1, l) B_h[..., l]
// For H1 this merges the reference's T = 10 final-stage terms
// (_kernels.py:604-621) into 4, for H(curl) its T = 5 (_kernels.py:1125-1147)
// into 1..4 per block pair, for H(div) its T = 2 (_kernels.py:838-850) into
// 1..2.
#pragma once
#include <stdint.h>

namespace hxg {

enum Space : int { H1 = 0, HCURL = 1, HDIV = 2, L2 = 3 };
enum Path : int { GENERAL = 0, AFFINE = 1, EXTRUSION = 2 };

// 1D table block layout (doubles), built by hxg_make_tables
constexpr int KT = 16;   // 1D function index capacity (k <= 15, p <= 12 needs k <= 13)
constexpr int LT = 16;   // quadrature-point capacity
constexpr int TAB_NODES = 0;
constexpr int TAB_WTS = TAB_NODES + LT;
constexpr int TAB_T = TAB_WTS + LT;             // T[f][k][l], f: 0 chi, 1 chi'
constexpr int TAB_F = TAB_T + 2 * KT * LT;      // F[rs][i][j], rs = 2r + s (poly1d.py:265)
constexpr int TAB_TOTAL = TAB_F + 4 * KT * KT;

constexpr int MAXT = 10;  // stage-A terms per block pair
constexpr int MAXG = 9;   // stage-B groups per block pair
constexpr int MAXH = 4;   // stage-C groups per block pair
constexpr int MAXF = 12;  // metric fields per point

struct PairPlan {
    int8_t nt, ng, nh, kdim_pad;
    int8_t t_g[MAXT], t_field[MAXT], t_fr[MAXT], t_fs[MAXT], t_sign[MAXT];
    int8_t g_h[MAXG], g_fr[MAXG], g_fs[MAXG];
    int8_t h_fr[MAXH], h_fs[MAXH];
};

struct SpacePlan {
    int space, nb, N, nfields;
    int n[3][3];      // extents n[a][d]
    int sh[3][3];     // 1D index shift of (block a, direction d)
    int off[3];       // block offsets in the flat index
    PairPlan pair[3][3];
};

// symmetric 3x3 index: 00 0, 11 1, 22 2, 01 3, 02 4, 12 5
__host__ __device__ inline int sym3(int a, int b)
{
    if (a == b) return a;
    int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo == 0 ? (hi == 1 ? 3 : 4) : 5;
}

}  // namespace hxg
