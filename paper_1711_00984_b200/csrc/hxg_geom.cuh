// hxg_geom.cuh -- per-point element geometry on the device (restatement of
// /root/reference/pkg/src/hexgram/_kernels.py:56-136) and the term fields of
// hxg_plan.h.  Inline device functions only (shared by several translation units).
#pragma once
#include "hxg_common.cuh"

namespace hxg {

// ---------------------------------------------------------------------------
// geometry (device restatement of _kernels.py:56-136)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dev_jacobian(int kind, const double *__restrict__ par, double x1,
                                             double x2, double x3, double J[3][3])
{
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) J[r][c] = 0.0;
    if (kind == 0) {
        J[0][0] = J[1][1] = J[2][2] = 1.0;
    } else if (kind == 1) {
        J[0][0] = par[0];
        J[1][1] = par[1];
        J[2][2] = par[2];
    } else if (kind == 2) {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) J[r][c] = par[3 * r + c];
    } else if (kind == 3) {
        J[0][0] = par[0];
        J[1][1] = (par[4] - par[2]) * (1.0 - x3) + (par[8] - par[6]) * x3;
        J[2][1] = (par[5] - par[3]) * (1.0 - x3) + (par[9] - par[7]) * x3;
        J[1][2] = (par[6] - par[2]) * (1.0 - x2) + (par[8] - par[4]) * x2;
        J[2][2] = (par[7] - par[3]) * (1.0 - x2) + (par[9] - par[5]) * x2;
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double f1 = (k & 1) ? x1 : 1.0 - x1;
            const double f2 = (k & 2) ? x2 : 1.0 - x2;
            const double f3 = (k & 4) ? x3 : 1.0 - x3;
            const double g1 = (k & 1) ? 1.0 : -1.0;
            const double g2 = (k & 2) ? 1.0 : -1.0;
            const double g3 = (k & 4) ? 1.0 : -1.0;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const double v = par[3 * k + r];
                J[r][0] += v * (g1 * f2 * f3);
                J[r][1] += v * (f1 * g2 * f3);
                J[r][2] += v * (f1 * f2 * g3);
            }
        }
    }
}

// det J, D = J^-1 J^-T (symmetric, sym3 order), C = J^T J (sym3 order)
__device__ __forceinline__ double dev_metrics(const double J[3][3], double D[6], double C[6])
{
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
    const int A[6] = {0, 1, 2, 0, 0, 1}, B[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int s = 0; s < 6; ++s) {
        const int a = A[s], b = B[s];
        D[s] = Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2];
        C[s] = J[0][a] * J[0][b] + J[1][a] * J[1][b] + J[2][a] * J[2][b];
    }
    return det;
}

// Term fields of hxg_plan.h for one point; w = quadrature weight, c = mass weight.
__device__ __forceinline__ int dev_fields(int space, double det, const double D[6],
                                          const double C[6], double w, double c, double f[MAXF])
{
    switch (space) {
    case H1:  // (c phi phi + grad D grad) det w   (_kernels.py:578-590)
        f[0] = c * det * w;
#pragma unroll
        for (int s = 0; s < 6; ++s) f[1 + s] = D[s] * det * w;
        return 7;
    case L2:  // c v v / det w                       (_kernels.py:389)
        f[0] = c * w / det;
        return 1;
    case HDIV:  // (c th C th + div div) / det w     (_kernels.py:781-797)
#pragma unroll
        for (int s = 0; s < 6; ++s) f[s] = c * C[s] * w / det;
        f[6] = w / det;
        return 7;
    default:  // Hcurl: c ps D ps det + curl C curl / det  (_kernels.py:1041-1068)
#pragma unroll
        for (int s = 0; s < 6; ++s) f[s] = c * D[s] * det * w;
#pragma unroll
        for (int s = 0; s < 6; ++s) f[6 + s] = C[s] * w / det;
        return 12;
    }
}

}  // namespace hxg
