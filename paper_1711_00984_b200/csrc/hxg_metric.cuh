// hxg_metric.cuh -- compile-time specialized per-point metric kernel (space S,
// rule size L): the term fields of hxg_plan.h at every quadrature point of every
// element (restatement of _kernels.py:56-136 plus the weight folding of
// _kernels.py:389, 578-590, 781-797, 1041-1068), for the general-map contraction.
//
// One warp per element: the element's map parameters are loaded once, the
// trilinear Jacobian is evaluated from the 12 edge-difference vectors (each
// column of J is a bilinear interpolation of 4 of them: 9 lerps per point instead
// of the 72-term vertex sum), the lanes run along the fastest index m of the
// metric layout [e][field][n][l][m] (coalesced stores), and the element's status
// word is written whole (bit 0: det J <= 0 somewhere), so no memset precedes it --
// or, when another kernel has flagged the word first (extrusion kind check),
// bit 0 is ORed in.
#pragma once
#include "hxg_geom.cuh"
#include "hxg_terms.h"

namespace hxg {

constexpr int MET2_WARPS = 8;

template <int S, int L>
__global__ void __launch_bounds__(MET2_WARPS * 32)
    metric_v2_kernel(int E, const int *__restrict__ kind, const double *__restrict__ params,
                     const double *__restrict__ coef, const double *__restrict__ wgrid,
                     const double *__restrict__ tab, double *__restrict__ metric, int *__restrict__ status,
                     int status_or)
{
    constexpr int L3 = L * L * L, NF = nf_of(S);
    const int lane = threadIdx.x & 31;
    const int e = blockIdx.x * MET2_WARPS + (threadIdx.x >> 5);
    if (e >= E) return;
    const int knd = kind[e];
    const double *par = params + 24LL * e;
    const double pv = lane < 24 ? par[lane] : 0.0;
    // edge differences of the trilinear map, vertex k <-> corner (k & 1, k >> 1 & 1, k >> 2 & 1)
    // (geometry.py:115-119): d[c][q][r] = v(corner with bit c set) - v(bit c clear), q = the
    // other two bits (low, high) in order
    double d[3][4][3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int lo = c == 0 ? 1 : 0, hi = c == 2 ? 1 : 2;  // the other two bit positions
            const int k0 = ((q & 1) << lo) | ((q >> 1) << hi), k1 = k0 | (1 << c);
#pragma unroll
            for (int r = 0; r < 3; ++r)
                d[c][q][r] = __shfl_sync(0xffffffffu, pv, 3 * k1 + r) - __shfl_sync(0xffffffffu, pv, 3 * k0 + r);
        }
    const double cf = coef ? coef[e] : 1.0;
    double *mo = metric + (long long)e * NF * L3;
    bool bad = false;
    for (int pt = lane; pt < L3; pt += 32) {
        const int n = pt / (L * L), l = (pt / L) % L, m = pt % L;
        const double x1 = tab[TAB_NODES + l], x2 = tab[TAB_NODES + m], x3 = tab[TAB_NODES + n];
        double J[3][3];
        if (knd == 4) {
            const double xs[3] = {x1, x2, x3};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double s = xs[c == 0 ? 1 : 0], t = xs[c == 2 ? 1 : 2];
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const double a = fma(s, d[c][1][r] - d[c][0][r], d[c][0][r]);
                    const double b = fma(s, d[c][3][r] - d[c][2][r], d[c][2][r]);
                    J[r][c] = fma(t, b - a, a);
                }
            }
        } else {
            dev_jacobian(knd, par, x1, x2, x3, J);
        }
        double D[6], C[6], f[MAXF];
        const double det = dev_metrics(J, D, C);
        const double w = tab[TAB_WTS + l] * tab[TAB_WTS + m] * tab[TAB_WTS + n];
        const double c = wgrid ? wgrid[(long long)e * L3 + (l * L + m) * L + n] : cf;
        dev_fields(S, det, D, C, w, c, f);
#pragma unroll
        for (int k = 0; k < NF; ++k) mo[k * L3 + pt] = f[k];
        bad |= !(det > 0.0);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) status[e] = (status_or ? status[e] : 0) | (bad ? 1 : 0);  // this warp owns word e
}

}  // namespace hxg
