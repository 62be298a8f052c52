// hxg_terms.h -- compile-time (constexpr) description of every space: block
// extents, 1D index shifts, integrand terms and their stage groups.
//
// Single source of truth for the host planner (hxg_capi.cu) and the
// specialized kernels (hxg_general_v2.cuh).  See hxg_plan.h for the term /
// group model.  Reference: spaces.py:95-102 (per-component digit ranges),
// shape3_eval spaces.py:161-232 (which 1D factor each component carries),
// _kernels.py:578-590, 781-797, 1041-1068 (per-point weights of each term).
#pragma once
#include "hxg_plan.h"

namespace hxg {

__host__ __device__ constexpr int nb_of(int S) { return (S == H1 || S == L2) ? 1 : 3; }

__host__ __device__ constexpr int nf_of(int S)
{
    return S == H1 ? 7 : S == L2 ? 1 : S == HDIV ? 7 : 12;
}

// digits of block a in direction d for order p_d
__host__ __device__ constexpr int ext_of(int S, int pd, int a, int d)
{
    return S == H1 ? pd + 1 : S == L2 ? pd : S == HDIV ? (d == a ? pd + 1 : pd) : (d == a ? pd : pd + 1);
}

// 1D table index = digit + shift (nu_i = chi'_{i+1})
__host__ __device__ constexpr int sh_of(int S, int a, int d)
{
    return S == H1 ? 0 : S == L2 ? 1 : S == HDIV ? (d == a ? 0 : 1) : (d == a ? 1 : 0);
}

// function code of the "value" factor: 0 chi, 1 chi'
__host__ __device__ constexpr int prim_of(int S, int a, int d)
{
    return S == H1 ? 0 : S == L2 ? 1 : S == HDIV ? (d == a ? 0 : 1) : (d == a ? 1 : 0);
}

__host__ __device__ constexpr int csym3(int a, int b)
{
    return a == b ? a : ((a < b ? a : b) == 0 ? (((a < b ? b : a) == 1) ? 3 : 4) : 5);
}

struct CPair {
    int nt, ng, nh;
    int t_g[MAXT], t_field[MAXT], t_fr[MAXT], t_fs[MAXT], t_sign[MAXT];
    int g_h[MAXG], g_fr[MAXG], g_fs[MAXG];
    int h_fr[MAXH], h_fs[MAXH];
    // distinct test-side xi1 function codes (Y-form stage C): nr <= 2
    int nr, r_code[2], h_r[MAXH];
};

// Terms of block pair (a, b) of space S, grouped for sum factorization.
__host__ __device__ constexpr CPair make_pair_plan(int S, int a, int b)
{
    CPair pp{};
    int tf[MAXT] = {}, ts[MAXT] = {};
    int fr[MAXT][3] = {}, fs[MAXT][3] = {};
    int n = 0;
    auto add = [&](int field, int sign, int r0, int r1, int r2, int s0, int s1, int s2) {
        tf[n] = field;
        ts[n] = sign;
        const int r[3] = {r0, r1, r2}, s[3] = {s0, s1, s2};
        for (int d = 0; d < 3; ++d) {
            fr[n][d] = r[d] ? 1 : prim_of(S, a, d);
            fs[n][d] = s[d] ? 1 : prim_of(S, b, d);
        }
        ++n;
    };
    if (S == H1) {  // (c phi phi + grad^T D grad) det
        add(0, 1, 0, 0, 0, 0, 0, 0);
        for (int al = 0; al < 3; ++al)
            for (int be = 0; be < 3; ++be)
                add(1 + csym3(al, be), 1, al == 0, al == 1, al == 2, be == 0, be == 1, be == 2);
    } else if (S == L2) {  // c v v / det
        add(0, 1, 0, 0, 0, 0, 0, 0);
    } else if (S == HDIV) {  // (c th^T C th + div div) / det
        add(csym3(a, b), 1, 0, 0, 0, 0, 0, 0);
        add(6, 1, a == 0, a == 1, a == 2, b == 0, b == 1, b == 2);
    } else {  // Hcurl: c ps^T D ps det + curl^T C curl / det
        add(csym3(a, b), 1, 0, 0, 0, 0, 0, 0);
        for (int al = 0; al < 2; ++al)
            for (int be = 0; be < 2; ++be) {
                const int ca = (a + al + 1) % 3, cb = (b + be + 1) % 3;
                add(6 + csym3(ca, cb), al == be ? 1 : -1,
                    0 != a && 0 != ca, 1 != a && 1 != ca, 2 != a && 2 != ca,
                    0 != b && 0 != cb, 1 != b && 1 != cb, 2 != b && 2 != cb);
            }
    }
    // g = (xi1 pair, xi2 pair), h = xi1 pair, in first-appearance order
    int gkey[MAXG] = {}, tg[MAXT] = {};
    int ng = 0;
    for (int t = 0; t < n; ++t) {
        const int k = ((fr[t][0] * 2 + fs[t][0]) * 2 + fr[t][1]) * 2 + fs[t][1];
        int g = -1;
        for (int q = 0; q < ng; ++q)
            if (gkey[q] == k) g = q;
        if (g < 0) { gkey[ng] = k; g = ng++; }
        tg[t] = g;
    }
    int hkey[MAXH] = {};
    int nh = 0;
    for (int g = 0; g < ng; ++g) {
        const int k = gkey[g] >> 2;
        int h = -1;
        for (int q = 0; q < nh; ++q)
            if (hkey[q] == k) h = q;
        if (h < 0) { hkey[nh] = k; h = nh++; }
        pp.g_h[g] = h;
        pp.g_fr[g] = (gkey[g] >> 1) & 1;
        pp.g_fs[g] = gkey[g] & 1;
    }
    for (int h = 0; h < nh; ++h) {
        pp.h_fr[h] = (hkey[h] >> 1) & 1;
        pp.h_fs[h] = hkey[h] & 1;
        int r = -1;
        for (int q = 0; q < pp.nr; ++q)
            if (pp.r_code[q] == pp.h_fr[h]) r = q;
        if (r < 0) { pp.r_code[pp.nr] = pp.h_fr[h]; r = pp.nr++; }
        pp.h_r[h] = r;
    }
    int k = 0;
    for (int g = 0; g < ng; ++g)
        for (int t = 0; t < n; ++t)
            if (tg[t] == g) {
                pp.t_g[k] = g;
                pp.t_field[k] = tf[t];
                pp.t_fr[k] = fr[t][2];
                pp.t_fs[k] = fs[t][2];
                pp.t_sign[k] = ts[t];
                ++k;
            }
    pp.nt = n;
    pp.ng = ng;
    pp.nh = nh;
    return pp;
}

}  // namespace hxg
