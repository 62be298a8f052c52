/*
 * hexgram_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99 + pthreads) of the reference package's Gram
 * integration hot path, used as the parity checker for the sm_100a kernels
 * and as the "port" CPU baseline in bench.py.  Nothing in the product path
 * (paper_1711_00984_b200/) links, imports or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu/reference legs do.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py, run in the build container where
 * /root/reference is importable).
 *
 * Reference citations are /root/reference/pkg/src/hexgram/<file>:<line>.
 * The restatement keeps the reference's *alternative* loop order
 * (quadrature loops outermost, _kernels.py:406-454, 541-624, 742-853,
 * 1003-1150), the simplified constant-Jacobian kernels
 * (_kernels.py:1169-1404) and the simplified extrusion kernels
 * (_kernels.py:1405-1764); both loop orders of the reference produce
 * bit-identical matrices (pkg/tests/test_gram.py:103-112).
 *
 * Output convention of the batched entry: per element, the packed upper
 * triangle in row-major order (LAPACK 'L' packed of the symmetric matrix):
 *   packed[r*N - r*(r-1)/2 + (c-r)] = G[r][c],  r <= c.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>
#include <pthread.h>
#include <unistd.h>

enum { ORC_H1 = 0, ORC_HCURL = 1, ORC_HDIV = 2, ORC_L2 = 3 };
enum { ORC_GENERAL = 0, ORC_AFFINE = 1, ORC_EXTRUSION = 2 };

/* ------------------------------------------------------------------ */
/* 1D machinery                                                         */
/* ------------------------------------------------------------------ */

/* quadrature.py:37-44 -- P_L and P_L' on [-1,1] by the 3-term recursion */
static void leg_pl(int L, double x, double *p_out, double *dp_out)
{
    double pm = 1.0, pc = x;
    for (int k = 2; k <= L; ++k) {
        double pn = ((2 * k - 1) * x * pc - (k - 1) * pm) / k;
        pm = pc;
        pc = pn;
    }
    *p_out = pc;
    *dp_out = L * (x * pc - pm) / (x * x - 1.0);
}

/* quadrature.py:47-66 -- Gauss-Legendre on (0,1), nodes increasing.
 * Newton iterations run on the whole node vector and stop when the
 * largest update is below 1e-15, as the reference does. */
int orc_gauss_rule(int L, double *nodes, double *weights)
{
    if (L < 1 || L > 32) return -1;
    if (L == 1) { nodes[0] = 0.5; weights[0] = 1.0; return 0; }
    double x[32];
    for (int k = 1; k <= L; ++k) x[k - 1] = cos(M_PI * (k - 0.25) / (L + 0.5));
    for (int it = 0; it < 100; ++it) {
        double mx = 0.0;
        double dx[32];
        for (int k = 0; k < L; ++k) {
            double p, dp;
            leg_pl(L, x[k], &p, &dp);
            dx[k] = p / dp;
        }
        for (int k = 0; k < L; ++k) {
            x[k] -= dx[k];
            if (fabs(dx[k]) > mx) mx = fabs(dx[k]);
        }
        if (mx < 1e-15) break;
    }
    for (int k = 0; k < L; ++k) {
        double p, dp;
        leg_pl(L, x[k], &p, &dp);
        double w = 2.0 / ((1.0 - x[k] * x[k]) * dp * dp);
        nodes[L - 1 - k] = 0.5 * (1.0 + x[k]);
        weights[L - 1 - k] = 0.5 * w;
    }
    return 0;
}

/* _kernels.py:29-43 -- chi_0..chi_p and chi'_0..chi'_p at xi */
void orc_shape1_h1(double xi, int p, double *chi, double *dchi)
{
    double t = 2.0 * xi - 1.0;
    chi[0] = 1.0 - xi;
    chi[1] = xi;
    dchi[0] = -1.0;
    dchi[1] = 1.0;
    double pm2 = 1.0, pm1 = t;
    for (int i = 2; i <= p; ++i) {
        double pi = ((2 * i - 1) * t * pm1 - (i - 1) * pm2) / i;
        chi[i] = (pi - pm2) / (2.0 * (2 * i - 1));
        dchi[i] = pm1;
        pm2 = pm1;
        pm1 = pi;
    }
}

/* _kernels.py:46-53 -- nu_0..nu_{p-1} (shifted Legendre) at xi */
void orc_shape1_l2(double xi, int p, double *nu)
{
    double t = 2.0 * xi - 1.0;
    nu[0] = 1.0;
    if (p >= 2) nu[1] = t;
    for (int i = 2; i < p; ++i)
        nu[i] = ((2 * i - 1) * t * nu[i - 1] - (i - 1) * nu[i - 2]) / i;
}

/* poly1d.py:140-175 -- closed-form integral of chi_i chi_j */
static double f00(int i, int j)
{
    if (i < j) { int t = i; i = j; j = t; }
    if (j >= 2) {
        if (i == j) return (1.0 / (2 * j + 1) + 1.0 / (2 * j - 3)) / (4.0 * (2 * j - 1) * (2 * j - 1));
        if (i == j + 2) return -1.0 / (4.0 * (2 * j + 3) * (2 * j - 1) * (2 * j + 1));
        return 0.0;
    }
    if (j == 1) {
        switch (i) { case 1: return 1.0 / 3.0; case 2: return -1.0 / 12.0; case 3: return -1.0 / 60.0; }
        return 0.0;
    }
    switch (i) { case 0: return 1.0 / 3.0; case 1: return 1.0 / 6.0; case 2: return -1.0 / 12.0; case 3: return 1.0 / 60.0; }
    return 0.0;
}

/* poly1d.py:178-198 -- closed-form integral of chi_i chi_j' */
static double f01(int i, int j)
{
    if (j == 0) return -f01(i, 1);
    if (i == 0) return j == 1 ? 0.5 : (j == 2 ? -1.0 / 6.0 : 0.0);
    if (i == 1) return j == 1 ? 0.5 : (j == 2 ? 1.0 / 6.0 : 0.0);
    if (i == 2) return j == 1 ? -1.0 / 6.0 : (j == 3 ? 1.0 / 30.0 : 0.0);
    if (j == i + 1) return 1.0 / (2.0 * (2 * i - 1) * (2 * i + 1));
    if (j == i - 1) return -1.0 / (2.0 * (2 * i - 1) * (2 * i - 3));
    return 0.0;
}

/* poly1d.py:201-210 -- closed-form integral of chi_i' chi_j' */
static double f11(int i, int j)
{
    if (i < j) { int t = i; i = j; j = t; }
    if (j >= 1) return i == j ? 1.0 / (2 * i - 1) : 0.0;
    if (i == 0) return 1.0;
    if (i == 1) return -1.0;
    return 0.0;
}

/* poly1d.py:251-266 -- stacked [F00, F01, F10 = F01^T, F11], (4, P+1, P+1) */
int orc_ftable(int pmax, double *fall)
{
    if (pmax < 1) return -1;
    int n = pmax + 1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            fall[0 * n * n + i * n + j] = f00(i, j);
            fall[1 * n * n + i * n + j] = f01(i, j);
            fall[2 * n * n + i * n + j] = f01(j, i);
            fall[3 * n * n + i * n + j] = f11(i, j);
        }
    return 0;
}

/* ------------------------------------------------------------------ */
/* geometry                                                             */
/* ------------------------------------------------------------------ */

/* _kernels.py:56-97 -- Jacobian J[r][c] = d x_r / d xi_c for kinds 0..4 */
static void geom_jac(int kind, const double *par, double x1, double x2, double x3, double J[3][3])
{
    memset(J, 0, 9 * sizeof(double));
    switch (kind) {
    case 0:
        J[0][0] = J[1][1] = J[2][2] = 1.0;
        break;
    case 1:
        J[0][0] = par[0]; J[1][1] = par[1]; J[2][2] = par[2];
        break;
    case 2:
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) J[r][c] = par[3 * r + c];
        break;
    case 3:
        J[0][0] = par[0];
        J[1][1] = (par[4] - par[2]) * (1.0 - x3) + (par[8] - par[6]) * x3;
        J[2][1] = (par[5] - par[3]) * (1.0 - x3) + (par[9] - par[7]) * x3;
        J[1][2] = (par[6] - par[2]) * (1.0 - x2) + (par[8] - par[4]) * x2;
        J[2][2] = (par[7] - par[3]) * (1.0 - x2) + (par[9] - par[5]) * x2;
        break;
    default:
        for (int k = 0; k < 8; ++k) {
            int b1 = k & 1, b2 = (k >> 1) & 1, b3 = (k >> 2) & 1;
            double f1 = b1 ? x1 : 1.0 - x1, f2 = b2 ? x2 : 1.0 - x2, f3 = b3 ? x3 : 1.0 - x3;
            double g1 = b1 ? 1.0 : -1.0, g2 = b2 ? 1.0 : -1.0, g3 = b3 ? 1.0 : -1.0;
            for (int r = 0; r < 3; ++r) {
                double v = par[3 * k + r];
                J[r][0] += v * g1 * f2 * f3;
                J[r][1] += v * f1 * g2 * f3;
                J[r][2] += v * f1 * f2 * g3;
            }
        }
    }
}

/* _kernels.py:100-118 -- cofactor inverse; returns det J */
double orc_geom_full(int kind, const double *par, double x1, double x2, double x3,
                     double J[3][3], double Ji[3][3])
{
    geom_jac(kind, par, x1, x2, x3, J);
    double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    double inv = 1.0 / det;
    Ji[0][0] = c00 * inv;
    Ji[1][0] = c01 * inv;
    Ji[2][0] = c02 * inv;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * inv;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * inv;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * inv;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * inv;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * inv;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * inv;
    return det;
}

/* _kernels.py:121-129 -- D = J^-1 J^-T */
static void metric_d(double Ji[3][3], double D[3][3])
{
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            D[a][b] = Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2];
}

/* _kernels.py:132-136 -- C = J^T J */
static void metric_c(double J[3][3], double C[3][3])
{
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            C[a][b] = J[0][a] * J[0][b] + J[1][a] * J[1][b] + J[2][a] * J[2][b];
}

/* ------------------------------------------------------------------ */
/* index maps (spaces.py:9-17, _kernels.py:139-158)                     */
/* ------------------------------------------------------------------ */

int orc_dim(int space, int p1, int p2, int p3)
{
    switch (space) {
    case ORC_H1: return (p1 + 1) * (p2 + 1) * (p3 + 1);
    case ORC_L2: return p1 * p2 * p3;
    case ORC_HDIV: return (p1 + 1) * p2 * p3 + p1 * (p2 + 1) * p3 + p1 * p2 * (p3 + 1);
    case ORC_HCURL: return p1 * (p2 + 1) * (p3 + 1) + (p1 + 1) * p2 * (p3 + 1) + (p1 + 1) * (p2 + 1) * p3;
    }
    return -1;
}

static int flat_hdiv(int a, int i1, int i2, int i3, int p1, int p2, int p3)
{
    if (a == 0) return i1 + (p1 + 1) * (i2 + p2 * i3);
    int off = (p1 + 1) * p2 * p3;
    if (a == 1) return off + i1 + p1 * (i2 + (p2 + 1) * i3);
    off += p1 * (p2 + 1) * p3;
    return off + i1 + p1 * (i2 + p2 * i3);
}

static int flat_hcurl(int a, int i1, int i2, int i3, int p1, int p2, int p3)
{
    if (a == 0) return i1 + p1 * (i2 + (p2 + 1) * i3);
    int off = p1 * (p2 + 1) * (p3 + 1);
    if (a == 1) return off + i1 + (p1 + 1) * (i2 + p2 * i3);
    off += (p1 + 1) * p2 * (p3 + 1);
    return off + i1 + (p1 + 1) * (i2 + (p2 + 1) * i3);
}

/* _kernels.py:169-174: copy the lower triangle onto the upper one */
static void mirror_lower(double *G, int N)
{
    for (int j = 0; j < N; ++j)
        for (int i = j + 1; i < N; ++i) G[(size_t)j * N + i] = G[(size_t)i * N + j];
}

/* _kernels.py:177-198: complete the L2 matrix from the coordinate-sorted
 * digit pairs (per-coordinate swap symmetry of the L2 integrand) */
static void fill_l2_sym(double *G, int p1, int p2, int p3)
{
    int N = p1 * p2 * p3;
    for (int I = 0; I < N; ++I) {
        int i1 = I % p1, i2 = (I / p1) % p2, i3 = I / (p1 * p2);
        for (int Jf = 0; Jf <= I; ++Jf) {
            int j1 = Jf % p1, j2 = (Jf / p1) % p2, j3 = Jf / (p1 * p2);
            int a1 = i1 >= j1 ? i1 : j1, b1 = i1 >= j1 ? j1 : i1;
            int a2 = i2 >= j2 ? i2 : j2, b2 = i2 >= j2 ? j2 : i2;
            int a3 = i3 >= j3 ? i3 : j3, b3 = i3 >= j3 ? j3 : i3;
            double v = G[(size_t)(a1 + p1 * (a2 + p2 * a3)) * N + (b1 + p1 * (b2 + p2 * b3))];
            G[(size_t)I * N + Jf] = v;
            G[(size_t)Jf * N + I] = v;
        }
    }
}

/* ------------------------------------------------------------------ */
/* tensorized kernels, alternative loop order                           */
/* wgrid[(l*L+m)*L+n] is the mass-term weight at the quadrature node.   */
/* Every function returns the accumulation count (OpCounters).          */
/* ------------------------------------------------------------------ */

/* _kernels.py:406-454 (tens_l2_alt) */
static long long tens_l2(int p1, int p2, int p3, int L, const double *nd, const double *wt,
                         int kind, const double *par, const double *wg, double *G)
{
    int N = p1 * p2 * p3;
    double nu1[64], nu2[64], nu3[64], J[3][3], Ji[3][3];
    double *gA = calloc((size_t)p3 * p3, sizeof(double));
    double *gB = calloc((size_t)p2 * p2 * p3 * p3, sizeof(double));
    long long acc = 0;
#define GB(i2, j2, i3, j3) gB[(((size_t)(i2) * p2 + (j2)) * p3 + (i3)) * p3 + (j3)]
    for (int l = 0; l < L; ++l) {
        orc_shape1_l2(nd[l], p1, nu1);
        memset(gB, 0, sizeof(double) * p2 * p2 * p3 * p3);
        for (int m = 0; m < L; ++m) {
            orc_shape1_l2(nd[m], p2, nu2);
            memset(gA, 0, sizeof(double) * p3 * p3);
            for (int n = 0; n < L; ++n) {
                orc_shape1_l2(nd[n], p3, nu3);
                double det = orc_geom_full(kind, par, nd[l], nd[m], nd[n], J, Ji);
                double c = wg[(l * L + m) * L + n] * wt[n] / det;
                for (int j3 = 0; j3 < p3; ++j3)
                    for (int i3 = j3; i3 < p3; ++i3) gA[i3 * p3 + j3] += nu3[i3] * nu3[j3] * c;
            }
            for (int j3 = 0; j3 < p3; ++j3)
                for (int i3 = j3; i3 < p3; ++i3)
                    for (int j2 = 0; j2 < p2; ++j2)
                        for (int i2 = j2; i2 < p2; ++i2)
                            GB(i2, j2, i3, j3) += nu2[i2] * nu2[j2] * gA[i3 * p3 + j3] * wt[m];
        }
        for (int j3 = 0; j3 < p3; ++j3)
            for (int i3 = j3; i3 < p3; ++i3)
                for (int j2 = 0; j2 < p2; ++j2)
                    for (int i2 = j2; i2 < p2; ++i2)
                        for (int j1 = 0; j1 < p1; ++j1)
                            for (int i1 = j1; i1 < p1; ++i1) {
                                int I = i1 + p1 * (i2 + p2 * i3), Jf = j1 + p1 * (j2 + p2 * j3);
                                G[(size_t)I * N + Jf] += nu1[i1] * nu1[j1] * GB(i2, j2, i3, j3) * wt[l];
                                ++acc;
                            }
    }
#undef GB
    fill_l2_sym(G, p1, p2, p3);
    free(gA);
    free(gB);
    return acc;
}

/* _kernels.py:541-624 (tens_h1_alt) */
static long long tens_h1(int p1, int p2, int p3, int L, const double *nd, const double *wt,
                         int kind, const double *par, const double *wg, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = q1 * q2 * q3;
    double c1[64], d1[64], c2[64], d2[64], c3[64], d3[64], J[3][3], Ji[3][3], D[3][3];
    size_t nA = (size_t)q3 * q3, nB = (size_t)q2 * q2 * q3 * q3;
    double *gAbar = malloc(nA * sizeof(double)), *gA = malloc(9 * nA * sizeof(double));
    double *gBbar = malloc(nB * sizeof(double)), *gB = malloc(9 * nB * sizeof(double));
    long long acc = 0;
#define IA(i3, j3) ((size_t)(i3) * q3 + (j3))
#define IB(i2, j2, i3, j3) ((((size_t)(i2) * q2 + (j2)) * q3 + (i3)) * q3 + (j3))
    for (int l = 0; l < L; ++l) {
        orc_shape1_h1(nd[l], p1, c1, d1);
        memset(gBbar, 0, nB * sizeof(double));
        memset(gB, 0, 9 * nB * sizeof(double));
        for (int m = 0; m < L; ++m) {
            orc_shape1_h1(nd[m], p2, c2, d2);
            memset(gAbar, 0, nA * sizeof(double));
            memset(gA, 0, 9 * nA * sizeof(double));
            for (int n = 0; n < L; ++n) {
                orc_shape1_h1(nd[n], p3, c3, d3);
                double det = orc_geom_full(kind, par, nd[l], nd[m], nd[n], J, Ji);
                metric_d(Ji, D);
                double wq = wt[n] * det, wm = wg[(l * L + m) * L + n] * wq;
                for (int j3 = 0; j3 < q3; ++j3)
                    for (int i3 = j3; i3 < q3; ++i3) {
                        gAbar[IA(i3, j3)] += c3[i3] * c3[j3] * wm;
                        for (int a = 0; a < 3; ++a) {
                            double fa = a == 2 ? d3[i3] : c3[i3];
                            for (int b = 0; b < 3; ++b) {
                                double fb = b == 2 ? d3[j3] : c3[j3];
                                gA[(a * 3 + b) * nA + IA(i3, j3)] += fa * fb * D[a][b] * wq;
                            }
                        }
                    }
            }
            for (int j3 = 0; j3 < q3; ++j3)
                for (int i3 = j3; i3 < q3; ++i3)
                    for (int j2 = 0; j2 < q2; ++j2)
                        for (int i2 = 0; i2 < q2; ++i2) {
                            gBbar[IB(i2, j2, i3, j3)] += c2[i2] * c2[j2] * gAbar[IA(i3, j3)] * wt[m];
                            for (int a = 0; a < 3; ++a) {
                                double fa = a == 1 ? d2[i2] : c2[i2];
                                for (int b = 0; b < 3; ++b) {
                                    double fb = b == 1 ? d2[j2] : c2[j2];
                                    gB[(a * 3 + b) * nB + IB(i2, j2, i3, j3)] +=
                                        fa * fb * gA[(a * 3 + b) * nA + IA(i3, j3)] * wt[m];
                                }
                            }
                        }
        }
        for (int j3 = 0; j3 < q3; ++j3)
            for (int i3 = j3; i3 < q3; ++i3)
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2)
                        for (int j1 = 0; j1 < q1; ++j1)
                            for (int i1 = 0; i1 < q1; ++i1) {
                                int I = i1 + q1 * (i2 + q2 * i3), Jf = j1 + q1 * (j2 + q2 * j3);
                                if (I < Jf) continue;
                                double val = c1[i1] * c1[j1] * gBbar[IB(i2, j2, i3, j3)];
                                ++acc;
                                for (int a = 0; a < 3; ++a) {
                                    double fa = a == 0 ? d1[i1] : c1[i1];
                                    for (int b = 0; b < 3; ++b) {
                                        double fb = b == 0 ? d1[j1] : c1[j1];
                                        val += fa * fb * gB[(a * 3 + b) * nB + IB(i2, j2, i3, j3)];
                                        ++acc;
                                    }
                                }
                                G[(size_t)I * N + Jf] += val * wt[l];
                            }
    }
#undef IA
#undef IB
    mirror_lower(G, N);
    free(gAbar); free(gA); free(gBbar); free(gB);
    return acc;
}

/* _kernels.py:742-853 (tens_hdiv_alt) */
static long long tens_hdiv(int p1, int p2, int p3, int L, const double *nd, const double *wt,
                           int kind, const double *par, const double *wg, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1;
    int N = orc_dim(ORC_HDIV, p1, p2, p3);
    double c1[64], d1[64], c2[64], d2[64], c3[64], d3[64], J[3][3], Ji[3][3], C[3][3];
    size_t nA = (size_t)q3 * q3, nB = (size_t)q2 * q2 * q3 * q3;
    double *gA = malloc(9 * nA * sizeof(double)), *gAt = malloc(9 * nA * sizeof(double));
    double *gB = malloc(9 * nB * sizeof(double)), *gBt = malloc(9 * nB * sizeof(double));
    long long acc = 0;
    int pp[3] = {p1, p2, p3};
#define IA(i3, j3) ((size_t)(i3) * q3 + (j3))
#define IB(i2, j2, i3, j3) ((((size_t)(i2) * q2 + (j2)) * q3 + (i3)) * q3 + (j3))
    for (int l = 0; l < L; ++l) {
        orc_shape1_h1(nd[l], p1, c1, d1);
        memset(gB, 0, 9 * nB * sizeof(double));
        memset(gBt, 0, 9 * nB * sizeof(double));
        for (int m = 0; m < L; ++m) {
            orc_shape1_h1(nd[m], p2, c2, d2);
            memset(gA, 0, 9 * nA * sizeof(double));
            memset(gAt, 0, 9 * nA * sizeof(double));
            for (int n = 0; n < L; ++n) {
                orc_shape1_h1(nd[n], p3, c3, d3);
                double det = orc_geom_full(kind, par, nd[l], nd[m], nd[n], J, Ji);
                metric_c(J, C);
                double wq = wt[n] / det, wm = wg[(l * L + m) * L + n] * wq;
                for (int j3 = 0; j3 < q3; ++j3)
                    for (int i3 = 0; i3 < q3; ++i3)
                        for (int a = 0; a < 3; ++a) {
                            int ia3 = a == 2 ? i3 : i3 + 1;
                            if (ia3 > p3) continue;
                            double fa = a == 2 ? c3[ia3] : d3[ia3];
                            for (int b = 0; b < 3; ++b) {
                                int jb3 = b == 2 ? j3 : j3 + 1;
                                if (jb3 > p3) continue;
                                double fb = b == 2 ? c3[jb3] : d3[jb3];
                                gA[(a * 3 + b) * nA + IA(i3, j3)] += fa * fb * C[a][b] * wm;
                                gAt[(a * 3 + b) * nA + IA(i3, j3)] += d3[ia3] * d3[jb3] * wq;
                            }
                        }
            }
            for (int j3 = 0; j3 < q3; ++j3)
                for (int i3 = 0; i3 < q3; ++i3)
                    for (int j2 = 0; j2 < q2; ++j2)
                        for (int i2 = 0; i2 < q2; ++i2)
                            for (int a = 0; a < 3; ++a) {
                                int ia2 = a == 1 ? i2 : i2 + 1;
                                if (ia2 > p2) continue;
                                double fa = a == 1 ? c2[ia2] : d2[ia2];
                                for (int b = 0; b < 3; ++b) {
                                    int jb2 = b == 1 ? j2 : j2 + 1;
                                    if (jb2 > p2) continue;
                                    double fb = b == 1 ? c2[jb2] : d2[jb2];
                                    size_t o = (a * 3 + b) * nB + IB(i2, j2, i3, j3);
                                    size_t oa = (a * 3 + b) * nA + IA(i3, j3);
                                    gB[o] += fa * fb * gA[oa] * wt[m];
                                    gBt[o] += d2[ia2] * d2[jb2] * gAt[oa] * wt[m];
                                }
                            }
        }
        for (int j3 = 0; j3 < q3; ++j3)
            for (int i3 = 0; i3 < q3; ++i3)
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2)
                        for (int j1 = 0; j1 < q1; ++j1)
                            for (int i1 = 0; i1 < q1; ++i1)
                                for (int a = 0; a < 3; ++a) {
                                    int ii[3] = {i1, i2, i3};
                                    int skip = 0;
                                    for (int d = 0; d < 3; ++d)
                                        if (d != a && ii[d] >= pp[d]) skip = 1;
                                    if (skip) continue;
                                    int ia1 = a == 0 ? i1 : i1 + 1;
                                    double fa = a == 0 ? c1[ia1] : d1[ia1];
                                    int I = flat_hdiv(a, i1, i2, i3, p1, p2, p3);
                                    for (int b = 0; b < 3; ++b) {
                                        int jj[3] = {j1, j2, j3};
                                        int skb = 0;
                                        for (int d = 0; d < 3; ++d)
                                            if (d != b && jj[d] >= pp[d]) skb = 1;
                                        if (skb) continue;
                                        int jb1 = b == 0 ? j1 : j1 + 1;
                                        int Jf = flat_hdiv(b, j1, j2, j3, p1, p2, p3);
                                        if (I < Jf) continue;
                                        double fb = b == 0 ? c1[jb1] : d1[jb1];
                                        size_t o = (a * 3 + b) * nB + IB(i2, j2, i3, j3);
                                        G[(size_t)I * N + Jf] += (fa * fb * gB[o] + d1[ia1] * d1[jb1] * gBt[o]) * wt[l];
                                        acc += 2;
                                    }
                                }
    }
#undef IA
#undef IB
    mirror_lower(G, N);
    free(gA); free(gAt); free(gB); free(gBt);
    return acc;
}

/* _kernels.py:1003-1150 (tens_hcurl_alt) */
static long long tens_hcurl(int p1, int p2, int p3, int L, const double *nd, const double *wt,
                            int kind, const double *par, const double *wg, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1;
    int N = orc_dim(ORC_HCURL, p1, p2, p3);
    double c1[64], d1[64], c2[64], d2[64], c3[64], d3[64], J[3][3], Ji[3][3], D[3][3], C[3][3];
    size_t nA = (size_t)q3 * q3, nB = (size_t)q2 * q2 * q3 * q3;
    /* gAc[a][b], gAa[al][be][a][b] (al, be in {0,1}) -- same layout for B */
    double *gAc = malloc(9 * nA * sizeof(double)), *gAa = malloc(36 * nA * sizeof(double));
    double *gBc = malloc(9 * nB * sizeof(double)), *gBa = malloc(36 * nB * sizeof(double));
    long long acc = 0;
    int pp[3] = {p1, p2, p3};
#define IA(i3, j3) ((size_t)(i3) * q3 + (j3))
#define IB(i2, j2, i3, j3) ((((size_t)(i2) * q2 + (j2)) * q3 + (i3)) * q3 + (j3))
#define CU(al, be, a, b) ((((al) * 2 + (be)) * 3 + (a)) * 3 + (b))
    for (int l = 0; l < L; ++l) {
        orc_shape1_h1(nd[l], p1, c1, d1);
        memset(gBc, 0, 9 * nB * sizeof(double));
        memset(gBa, 0, 36 * nB * sizeof(double));
        for (int m = 0; m < L; ++m) {
            orc_shape1_h1(nd[m], p2, c2, d2);
            memset(gAc, 0, 9 * nA * sizeof(double));
            memset(gAa, 0, 36 * nA * sizeof(double));
            for (int n = 0; n < L; ++n) {
                orc_shape1_h1(nd[n], p3, c3, d3);
                double det = orc_geom_full(kind, par, nd[l], nd[m], nd[n], J, Ji);
                metric_d(Ji, D);
                metric_c(J, C);
                double wqD = wt[n] * det * wg[(l * L + m) * L + n], wqC = wt[n] / det;
                for (int j3 = 0; j3 < q3; ++j3)
                    for (int i3 = 0; i3 < q3; ++i3)
                        for (int a = 0; a < 3; ++a) {
                            int ia3 = a == 2 ? i3 + 1 : i3;
                            if (ia3 > p3) continue;
                            double va = a == 2 ? d3[ia3] : c3[ia3];
                            for (int b = 0; b < 3; ++b) {
                                int jb3 = b == 2 ? j3 + 1 : j3;
                                if (jb3 > p3) continue;
                                double vb = b == 2 ? d3[jb3] : c3[jb3];
                                gAc[(a * 3 + b) * nA + IA(i3, j3)] += va * vb * D[a][b] * wqD;
                                for (int al = 0; al < 2; ++al) {
                                    int ca = (a + al + 1) % 3;
                                    double fa = ca == 2 ? c3[ia3] : d3[ia3];
                                    for (int be = 0; be < 2; ++be) {
                                        int cb = (b + be + 1) % 3;
                                        double fb = cb == 2 ? c3[jb3] : d3[jb3];
                                        gAa[CU(al, be, a, b) * nA + IA(i3, j3)] += fa * fb * C[ca][cb] * wqC;
                                    }
                                }
                            }
                        }
            }
            for (int j3 = 0; j3 < q3; ++j3)
                for (int i3 = 0; i3 < q3; ++i3)
                    for (int j2 = 0; j2 < q2; ++j2)
                        for (int i2 = 0; i2 < q2; ++i2)
                            for (int a = 0; a < 3; ++a) {
                                int ia2 = a == 1 ? i2 + 1 : i2;
                                if (ia2 > p2) continue;
                                double va = a == 1 ? d2[ia2] : c2[ia2];
                                for (int b = 0; b < 3; ++b) {
                                    int jb2 = b == 1 ? j2 + 1 : j2;
                                    if (jb2 > p2) continue;
                                    double vb = b == 1 ? d2[jb2] : c2[jb2];
                                    gBc[(a * 3 + b) * nB + IB(i2, j2, i3, j3)] +=
                                        va * vb * gAc[(a * 3 + b) * nA + IA(i3, j3)] * wt[m];
                                    for (int al = 0; al < 2; ++al) {
                                        int ca = (a + al + 1) % 3;
                                        double fa = ca == 1 ? c2[ia2] : d2[ia2];
                                        for (int be = 0; be < 2; ++be) {
                                            int cb = (b + be + 1) % 3;
                                            double fb = cb == 1 ? c2[jb2] : d2[jb2];
                                            gBa[CU(al, be, a, b) * nB + IB(i2, j2, i3, j3)] +=
                                                fa * fb * gAa[CU(al, be, a, b) * nA + IA(i3, j3)] * wt[m];
                                        }
                                    }
                                }
                            }
        }
        for (int j3 = 0; j3 < q3; ++j3)
            for (int i3 = 0; i3 < q3; ++i3)
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2)
                        for (int j1 = 0; j1 < q1; ++j1)
                            for (int i1 = 0; i1 < q1; ++i1)
                                for (int a = 0; a < 3; ++a) {
                                    int ii[3] = {i1, i2, i3};
                                    if (ii[a] >= pp[a]) continue;
                                    int ia1 = a == 0 ? i1 + 1 : i1;
                                    double va = a == 0 ? d1[ia1] : c1[ia1];
                                    int I = flat_hcurl(a, i1, i2, i3, p1, p2, p3);
                                    for (int b = 0; b < 3; ++b) {
                                        int jj[3] = {j1, j2, j3};
                                        if (jj[b] >= pp[b]) continue;
                                        int jb1 = b == 0 ? j1 + 1 : j1;
                                        int Jf = flat_hcurl(b, j1, j2, j3, p1, p2, p3);
                                        if (I < Jf) continue;
                                        double vb = b == 0 ? d1[jb1] : c1[jb1];
                                        double val = va * vb * gBc[(a * 3 + b) * nB + IB(i2, j2, i3, j3)];
                                        ++acc;
                                        for (int al = 0; al < 2; ++al) {
                                            int ca = (a + al + 1) % 3;
                                            double fa = ca == 0 ? c1[ia1] : d1[ia1];
                                            for (int be = 0; be < 2; ++be) {
                                                int cb = (b + be + 1) % 3;
                                                double fb = cb == 0 ? c1[jb1] : d1[jb1];
                                                double sgn = al == be ? 1.0 : -1.0;
                                                val += sgn * fa * fb * gBa[CU(al, be, a, b) * nB + IB(i2, j2, i3, j3)];
                                                ++acc;
                                            }
                                        }
                                        G[(size_t)I * N + Jf] += val * wt[l];
                                    }
                                }
    }
#undef IA
#undef IB
#undef CU
    mirror_lower(G, N);
    free(gAc); free(gAa); free(gBc); free(gBa);
    return acc;
}

/* ------------------------------------------------------------------ */
/* simplified kernels, constant-Jacobian maps (_kernels.py:1169-1404)  */
/* fall = stacked F tables (4, P+1, P+1), P = pmaxF                      */
/* ------------------------------------------------------------------ */
#define FT(rs, i, j) fall[((size_t)(rs) * nF + (i)) * nF + (j)]

/* _kernels.py:1169-1191 (simp_l2_const) */
static long long simp_l2(int p1, int p2, int p3, const double *fall, int nF, int kind,
                         const double *par, double wmass, double *G)
{
    int N = p1 * p2 * p3;
    double J[3][3], Ji[3][3];
    double det = orc_geom_full(kind, par, 0.5, 0.5, 0.5, J, Ji);
    long long acc = 0;
    for (int j3 = 0; j3 < p3; ++j3)
        for (int i3 = j3; i3 < p3; ++i3) {
            double gA = FT(3, i3 + 1, j3 + 1) * wmass / det;
            for (int j2 = 0; j2 < p2; ++j2)
                for (int i2 = j2; i2 < p2; ++i2) {
                    double gB = FT(3, i2 + 1, j2 + 1) * gA;
                    for (int j1 = 0; j1 < p1; ++j1)
                        for (int i1 = j1; i1 < p1; ++i1) {
                            int I = i1 + p1 * (i2 + p2 * i3), Jf = j1 + p1 * (j2 + p2 * j3);
                            G[(size_t)I * N + Jf] = FT(3, i1 + 1, j1 + 1) * gB;
                            ++acc;
                        }
                }
        }
    fill_l2_sym(G, p1, p2, p3);
    return acc;
}

/* _kernels.py:1194-1239 (simp_h1_const) with _rs_h1 (1160-1166) */
static long long simp_h1(int p1, int p2, int p3, const double *fall, int nF, int kind,
                         const double *par, double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = q1 * q2 * q3;
    double J[3][3], Ji[3][3], D[3][3];
    double det = orc_geom_full(kind, par, 0.5, 0.5, 0.5, J, Ji);
    metric_d(Ji, D);
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = j3; i3 < q3; ++i3)
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1) {
                            int I = i1 + q1 * (i2 + q2 * i3), Jf = j1 + q1 * (j2 + q2 * j3);
                            if (I < Jf) continue;
                            double val = wmass * FT(0, i1, j1) * FT(0, i2, j2) * FT(0, i3, j3);
                            ++acc;
                            for (int a = 0; a < 3; ++a)
                                for (int b = 0; b < 3; ++b) {
                                    int r1 = 2 * (a == 0) + (b == 0), r2 = 2 * (a == 1) + (b == 1), r3 = 2 * (a == 2) + (b == 2);
                                    val += D[a][b] * FT(r1, i1, j1) * FT(r2, i2, j2) * FT(r3, i3, j3);
                                    ++acc;
                                }
                            G[(size_t)I * N + Jf] += val * det;
                        }
    mirror_lower(G, N);
    return acc;
}

/* _kernels.py:1242-1310 (simp_hdiv_const) */
static long long simp_hdiv(int p1, int p2, int p3, const double *fall, int nF, int kind,
                           const double *par, double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = orc_dim(ORC_HDIV, p1, p2, p3);
    double J[3][3], Ji[3][3], C[3][3];
    double det = orc_geom_full(kind, par, 0.5, 0.5, 0.5, J, Ji);
    metric_c(J, C);
    int pp[3] = {p1, p2, p3};
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = 0; i3 < q3; ++i3)
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1)
                            for (int a = 0; a < 3; ++a) {
                                int ii[3] = {i1, i2, i3}, sk = 0;
                                for (int d = 0; d < 3; ++d) if (d != a && ii[d] >= pp[d]) sk = 1;
                                if (sk) continue;
                                int ia[3];
                                for (int d = 0; d < 3; ++d) ia[d] = d == a ? ii[d] : ii[d] + 1;
                                int I = flat_hdiv(a, i1, i2, i3, p1, p2, p3);
                                for (int b = 0; b < 3; ++b) {
                                    int jj[3] = {j1, j2, j3}, sb = 0;
                                    for (int d = 0; d < 3; ++d) if (d != b && jj[d] >= pp[d]) sb = 1;
                                    if (sb) continue;
                                    int jb[3];
                                    for (int d = 0; d < 3; ++d) jb[d] = d == b ? jj[d] : jj[d] + 1;
                                    int Jf = flat_hdiv(b, j1, j2, j3, p1, p2, p3);
                                    if (I < Jf) continue;
                                    double v = wmass * C[a][b];
                                    for (int d = 0; d < 3; ++d) {
                                        int rs = 2 * (d != a) + (d != b);
                                        v *= FT(rs, ia[d], jb[d]);
                                    }
                                    ++acc;
                                    v += FT(3, ia[0], jb[0]) * FT(3, ia[1], jb[1]) * FT(3, ia[2], jb[2]);
                                    ++acc;
                                    G[(size_t)I * N + Jf] += v / det;
                                }
                            }
    mirror_lower(G, N);
    return acc;
}

/* _kernels.py:1327-1404 (simp_hcurl_const) with _rs_hcurl_curl (1313-1324) */
static long long simp_hcurl(int p1, int p2, int p3, const double *fall, int nF, int kind,
                            const double *par, double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = orc_dim(ORC_HCURL, p1, p2, p3);
    double J[3][3], Ji[3][3], D[3][3], C[3][3];
    double det = orc_geom_full(kind, par, 0.5, 0.5, 0.5, J, Ji);
    metric_d(Ji, D);
    metric_c(J, C);
    int pp[3] = {p1, p2, p3};
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = 0; i3 < q3; ++i3)
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1)
                            for (int a = 0; a < 3; ++a) {
                                int ii[3] = {i1, i2, i3};
                                if (ii[a] >= pp[a]) continue;
                                int ia[3];
                                for (int d = 0; d < 3; ++d) ia[d] = d == a ? ii[d] + 1 : ii[d];
                                int I = flat_hcurl(a, i1, i2, i3, p1, p2, p3);
                                for (int b = 0; b < 3; ++b) {
                                    int jj[3] = {j1, j2, j3};
                                    if (jj[b] >= pp[b]) continue;
                                    int jb[3];
                                    for (int d = 0; d < 3; ++d) jb[d] = d == b ? jj[d] + 1 : jj[d];
                                    int Jf = flat_hcurl(b, j1, j2, j3, p1, p2, p3);
                                    if (I < Jf) continue;
                                    double val = wmass * D[a][b] * det;
                                    for (int d = 0; d < 3; ++d) {
                                        int rs = 2 * (d == a) + (d == b);
                                        val *= FT(rs, ia[d], jb[d]);
                                    }
                                    ++acc;
                                    for (int al = 0; al < 2; ++al)
                                        for (int be = 0; be < 2; ++be) {
                                            int ca = (a + al + 1) % 3, cb = (b + be + 1) % 3;
                                            double sgn = al == be ? 1.0 : -1.0;
                                            double t = sgn * C[ca][cb] / det;
                                            for (int d = 0; d < 3; ++d) {
                                                int rs = 2 * (d != ca) + (d != cb);
                                                t *= FT(rs, ia[d], jb[d]);
                                            }
                                            val += t;
                                            ++acc;
                                        }
                                    G[(size_t)I * N + Jf] += val;
                                }
                            }
    mirror_lower(G, N);
    return acc;
}

/* ------------------------------------------------------------------ */
/* simplified kernels, extrusion maps (_kernels.py:1405-1764):          */
/* quadrature in (xi2, xi3) at xi1 = 0.5, F-table factor in xi1          */
/* ------------------------------------------------------------------ */

/* _kernels.py:1412-1451 (simp_l2_ext) */
static long long simp_l2_ext(int p1, int p2, int p3, const double *fall, int nF, int L,
                             const double *nd, const double *wt, int kind, const double *par,
                             double wmass, double *G)
{
    int N = p1 * p2 * p3;
    double nu2[64], nu3[64], J[3][3], Ji[3][3];
    double *gB = malloc(sizeof(double) * p2 * p2);
    long long acc = 0;
    for (int j3 = 0; j3 < p3; ++j3)
        for (int i3 = j3; i3 < p3; ++i3) {
            for (int t = 0; t < p2 * p2; ++t) gB[t] = 0.0;
            for (int m = 0; m < L; ++m) {
                orc_shape1_l2(nd[m], p2, nu2);
                double gA = 0.0;
                for (int n = 0; n < L; ++n) {
                    orc_shape1_l2(nd[n], p3, nu3);
                    double detj = orc_geom_full(kind, par, 0.5, nd[m], nd[n], J, Ji);
                    gA += nu3[i3] * nu3[j3] * wmass * wt[n] / detj;
                }
                for (int j2 = 0; j2 < p2; ++j2)
                    for (int i2 = j2; i2 < p2; ++i2) gB[i2 * p2 + j2] += nu2[i2] * nu2[j2] * gA * wt[m];
            }
            for (int j2 = 0; j2 < p2; ++j2)
                for (int i2 = j2; i2 < p2; ++i2)
                    for (int j1 = 0; j1 < p1; ++j1)
                        for (int i1 = j1; i1 < p1; ++i1) {
                            int I = i1 + p1 * (i2 + p2 * i3), Jf = j1 + p1 * (j2 + p2 * j3);
                            G[(size_t)I * N + Jf] = FT(3, i1 + 1, j1 + 1) * gB[i2 * p2 + j2];
                            ++acc;
                        }
        }
    free(gB);
    fill_l2_sym(G, p1, p2, p3);
    return acc;
}

/* _kernels.py:1454-1531 (simp_h1_ext) with _rs_h1 (1160-1166) */
static long long simp_h1_ext(int p1, int p2, int p3, const double *fall, int nF, int L,
                             const double *nd, const double *wt, int kind, const double *par,
                             double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = q1 * q2 * q3;
    double chi2[64], dchi2[64], chi3[64], dchi3[64], J[3][3], Ji[3][3], D[3][3], gA[3][3];
    double *gBbar = malloc(sizeof(double) * q2 * q2);
    double *gB = malloc(sizeof(double) * 9 * q2 * q2);
#define GB(a, b, i, j) gB[(((a) * 3 + (b)) * q2 + (i)) * q2 + (j)]
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = j3; i3 < q3; ++i3) {
            for (int t = 0; t < q2 * q2; ++t) gBbar[t] = 0.0;
            for (int t = 0; t < 9 * q2 * q2; ++t) gB[t] = 0.0;
            for (int m = 0; m < L; ++m) {
                orc_shape1_h1(nd[m], p2, chi2, dchi2);
                double gAbar = 0.0;
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) gA[a][b] = 0.0;
                for (int n = 0; n < L; ++n) {
                    orc_shape1_h1(nd[n], p3, chi3, dchi3);
                    double detj = orc_geom_full(kind, par, 0.5, nd[m], nd[n], J, Ji);
                    metric_d(Ji, D);
                    double wq = wt[n] * detj;
                    gAbar += chi3[i3] * chi3[j3] * wmass * wq;
                    for (int a = 0; a < 3; ++a) {
                        double fa = a == 2 ? dchi3[i3] : chi3[i3];
                        for (int b = 0; b < 3; ++b) {
                            double fb = b == 2 ? dchi3[j3] : chi3[j3];
                            gA[a][b] += fa * fb * D[a][b] * wq;
                        }
                    }
                }
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2) {
                        gBbar[i2 * q2 + j2] += chi2[i2] * chi2[j2] * gAbar * wt[m];
                        for (int a = 0; a < 3; ++a) {
                            double fa = a == 1 ? dchi2[i2] : chi2[i2];
                            for (int b = 0; b < 3; ++b) {
                                double fb = b == 1 ? dchi2[j2] : chi2[j2];
                                GB(a, b, i2, j2) += fa * fb * gA[a][b] * wt[m];
                            }
                        }
                    }
            }
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1) {
                            int I = i1 + q1 * (i2 + q2 * i3), Jf = j1 + q1 * (j2 + q2 * j3);
                            if (I < Jf) continue;
                            double val = FT(0, i1, j1) * gBbar[i2 * q2 + j2];
                            ++acc;
                            for (int a = 0; a < 3; ++a)
                                for (int b = 0; b < 3; ++b) {
                                    int rs = 2 * (a == 0) + (b == 0);
                                    val += FT(rs, i1, j1) * GB(a, b, i2, j2);
                                    ++acc;
                                }
                            G[(size_t)I * N + Jf] += val;
                        }
        }
#undef GB
    free(gBbar);
    free(gB);
    mirror_lower(G, N);
    return acc;
}

/* _kernels.py:1534-1637 (simp_hdiv_ext) */
static long long simp_hdiv_ext(int p1, int p2, int p3, const double *fall, int nF, int L,
                               const double *nd, const double *wt, int kind, const double *par,
                               double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = orc_dim(ORC_HDIV, p1, p2, p3);
    double chi2[64], dchi2[64], chi3[64], dchi3[64], J[3][3], Ji[3][3], C[3][3];
    double gA[3][3], gAt[3][3];
    double *gB = malloc(sizeof(double) * 9 * q2 * q2);
    double *gBt = malloc(sizeof(double) * 9 * q2 * q2);
#define GB(x, a, b, i, j) x[(((a) * 3 + (b)) * q2 + (i)) * q2 + (j)]
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = 0; i3 < q3; ++i3) {
            for (int t = 0; t < 9 * q2 * q2; ++t) gB[t] = gBt[t] = 0.0;
            for (int m = 0; m < L; ++m) {
                orc_shape1_h1(nd[m], p2, chi2, dchi2);
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) gA[a][b] = gAt[a][b] = 0.0;
                for (int n = 0; n < L; ++n) {
                    orc_shape1_h1(nd[n], p3, chi3, dchi3);
                    double detj = orc_geom_full(kind, par, 0.5, nd[m], nd[n], J, Ji);
                    metric_c(J, C);
                    double wq = wt[n] / detj;
                    double wm = wmass * wq;
                    for (int a = 0; a < 3; ++a) {
                        int ia3 = a == 2 ? i3 : i3 + 1;
                        if (ia3 > p3) continue;
                        double fa = a == 2 ? chi3[ia3] : dchi3[ia3];
                        for (int b = 0; b < 3; ++b) {
                            int jb3 = b == 2 ? j3 : j3 + 1;
                            if (jb3 > p3) continue;
                            double fb = b == 2 ? chi3[jb3] : dchi3[jb3];
                            gA[a][b] += fa * fb * C[a][b] * wm;
                            gAt[a][b] += dchi3[ia3] * dchi3[jb3] * wq;
                        }
                    }
                }
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2)
                        for (int a = 0; a < 3; ++a) {
                            int ia2 = a == 1 ? i2 : i2 + 1;
                            if (ia2 > p2) continue;
                            double fa = a == 1 ? chi2[ia2] : dchi2[ia2];
                            for (int b = 0; b < 3; ++b) {
                                int jb2 = b == 1 ? j2 : j2 + 1;
                                if (jb2 > p2) continue;
                                double fb = b == 1 ? chi2[jb2] : dchi2[jb2];
                                GB(gB, a, b, i2, j2) += fa * fb * gA[a][b] * wt[m];
                                GB(gBt, a, b, i2, j2) += dchi2[ia2] * dchi2[jb2] * gAt[a][b] * wt[m];
                            }
                        }
            }
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1)
                            for (int a = 0; a < 3; ++a) {
                                if ((a != 0 && i1 >= p1) || (a != 1 && i2 >= p2) || (a != 2 && i3 >= p3)) continue;
                                int ia1 = a == 0 ? i1 : i1 + 1;
                                int I = flat_hdiv(a, i1, i2, i3, p1, p2, p3);
                                for (int b = 0; b < 3; ++b) {
                                    if ((b != 0 && j1 >= p1) || (b != 1 && j2 >= p2) || (b != 2 && j3 >= p3)) continue;
                                    int jb1 = b == 0 ? j1 : j1 + 1;
                                    int Jf = flat_hdiv(b, j1, j2, j3, p1, p2, p3);
                                    if (I >= Jf) {
                                        int rs = 2 * (a == 0 ? 0 : 1) + (b == 0 ? 0 : 1);
                                        G[(size_t)I * N + Jf] += FT(rs, ia1, jb1) * GB(gB, a, b, i2, j2) +
                                                                 FT(3, ia1, jb1) * GB(gBt, a, b, i2, j2);
                                        acc += 2;
                                    }
                                }
                            }
        }
#undef GB
    free(gB);
    free(gBt);
    mirror_lower(G, N);
    return acc;
}

/* _kernels.py:1640-1764 (simp_hcurl_ext) with _rs_hcurl_curl (1313-1324) */
static long long simp_hcurl_ext(int p1, int p2, int p3, const double *fall, int nF, int L,
                                const double *nd, const double *wt, int kind, const double *par,
                                double wmass, double *G)
{
    int q1 = p1 + 1, q2 = p2 + 1, q3 = p3 + 1, N = orc_dim(ORC_HCURL, p1, p2, p3);
    double chi2[64], dchi2[64], chi3[64], dchi3[64], J[3][3], Ji[3][3], D[3][3], C[3][3];
    double gAc[3][3], gAa[2][2][3][3];
    double *gBc = malloc(sizeof(double) * 9 * q2 * q2);
    double *gBa = malloc(sizeof(double) * 36 * q2 * q2);
#define GBC(a, b, i, j) gBc[(((a) * 3 + (b)) * q2 + (i)) * q2 + (j)]
#define GBA(al, be, a, b, i, j) gBa[(((((al) * 2 + (be)) * 3 + (a)) * 3 + (b)) * q2 + (i)) * q2 + (j)]
    long long acc = 0;
    for (int j3 = 0; j3 < q3; ++j3)
        for (int i3 = 0; i3 < q3; ++i3) {
            for (int t = 0; t < 9 * q2 * q2; ++t) gBc[t] = 0.0;
            for (int t = 0; t < 36 * q2 * q2; ++t) gBa[t] = 0.0;
            for (int m = 0; m < L; ++m) {
                orc_shape1_h1(nd[m], p2, chi2, dchi2);
                memset(gAc, 0, sizeof(gAc));
                memset(gAa, 0, sizeof(gAa));
                for (int n = 0; n < L; ++n) {
                    orc_shape1_h1(nd[n], p3, chi3, dchi3);
                    double detj = orc_geom_full(kind, par, 0.5, nd[m], nd[n], J, Ji);
                    metric_d(Ji, D);
                    metric_c(J, C);
                    double wqD = wt[n] * detj * wmass;
                    double wqC = wt[n] / detj;
                    for (int a = 0; a < 3; ++a) {
                        int ia3 = a == 2 ? i3 + 1 : i3;
                        if (ia3 > p3) continue;
                        double va = a == 2 ? dchi3[ia3] : chi3[ia3];
                        for (int b = 0; b < 3; ++b) {
                            int jb3 = b == 2 ? j3 + 1 : j3;
                            if (jb3 > p3) continue;
                            double vb = b == 2 ? dchi3[jb3] : chi3[jb3];
                            gAc[a][b] += va * vb * D[a][b] * wqD;
                            for (int al = 0; al < 2; ++al) {
                                int ca = (a + al + 1) % 3;
                                double fa = ca == 2 ? chi3[ia3] : dchi3[ia3];
                                for (int be = 0; be < 2; ++be) {
                                    int cb = (b + be + 1) % 3;
                                    double fb = cb == 2 ? chi3[jb3] : dchi3[jb3];
                                    gAa[al][be][a][b] += fa * fb * C[ca][cb] * wqC;
                                }
                            }
                        }
                    }
                }
                for (int j2 = 0; j2 < q2; ++j2)
                    for (int i2 = 0; i2 < q2; ++i2)
                        for (int a = 0; a < 3; ++a) {
                            int ia2 = a == 1 ? i2 + 1 : i2;
                            if (ia2 > p2) continue;
                            double va = a == 1 ? dchi2[ia2] : chi2[ia2];
                            for (int b = 0; b < 3; ++b) {
                                int jb2 = b == 1 ? j2 + 1 : j2;
                                if (jb2 > p2) continue;
                                double vb = b == 1 ? dchi2[jb2] : chi2[jb2];
                                GBC(a, b, i2, j2) += va * vb * gAc[a][b] * wt[m];
                                for (int al = 0; al < 2; ++al) {
                                    int ca = (a + al + 1) % 3;
                                    double fa = ca == 1 ? chi2[ia2] : dchi2[ia2];
                                    for (int be = 0; be < 2; ++be) {
                                        int cb = (b + be + 1) % 3;
                                        double fb = cb == 1 ? chi2[jb2] : dchi2[jb2];
                                        GBA(al, be, a, b, i2, j2) += fa * fb * gAa[al][be][a][b] * wt[m];
                                    }
                                }
                            }
                        }
            }
            for (int j2 = 0; j2 < q2; ++j2)
                for (int i2 = 0; i2 < q2; ++i2)
                    for (int j1 = 0; j1 < q1; ++j1)
                        for (int i1 = 0; i1 < q1; ++i1)
                            for (int a = 0; a < 3; ++a) {
                                if ((a == 0 && i1 >= p1) || (a == 1 && i2 >= p2) || (a == 2 && i3 >= p3)) continue;
                                int ia1 = a == 0 ? i1 + 1 : i1;
                                int I = flat_hcurl(a, i1, i2, i3, p1, p2, p3);
                                for (int b = 0; b < 3; ++b) {
                                    if ((b == 0 && j1 >= p1) || (b == 1 && j2 >= p2) || (b == 2 && j3 >= p3)) continue;
                                    int jb1 = b == 0 ? j1 + 1 : j1;
                                    int Jf = flat_hcurl(b, j1, j2, j3, p1, p2, p3);
                                    if (I >= Jf) {
                                        int rs = 2 * (a == 0 ? 1 : 0) + (b == 0 ? 1 : 0);
                                        double val = FT(rs, ia1, jb1) * GBC(a, b, i2, j2);
                                        ++acc;
                                        for (int al = 0; al < 2; ++al)
                                            for (int be = 0; be < 2; ++be) {
                                                double sgn = al == be ? 1.0 : -1.0;
                                                int ca = (a + al + 1) % 3, cb = (b + be + 1) % 3;
                                                int rc = 2 * (ca == 0 ? 0 : 1) + (cb == 0 ? 0 : 1);
                                                val += sgn * FT(rc, ia1, jb1) * GBA(al, be, a, b, i2, j2);
                                                ++acc;
                                            }
                                        G[(size_t)I * N + Jf] += val;
                                    }
                                }
                            }
        }
#undef GBC
#undef GBA
    free(gBc);
    free(gBa);
    mirror_lower(G, N);
    return acc;
}
#undef FT

/* ------------------------------------------------------------------ */
/* public entries                                                       */
/* ------------------------------------------------------------------ */

/* One element, full N x N matrix (what gram.py:139-158 / 161-205 return).
 * path 0: tensorized (gram_tensorized), wgrid[L^3] may be NULL (-> coef).
 * path 1: simplified constant-Jacobian (gram_simplified), kinds 0..2 only.
 * path 2: simplified extrusion (gram_simplified, simp_*_ext), kinds 0..3, rule L
 *         in (xi2, xi3).
 * Returns the accumulation counter, or -1 on a bad argument. */
long long orc_gram_full(int space, int path, int p1, int p2, int p3, int L,
                        const double *nodes, const double *weights,
                        int kind, const double *par, double coef, const double *wgrid,
                        double *G)
{
    int N = orc_dim(space, p1, p2, p3);
    if (N <= 0 || p1 < 1 || p2 < 1 || p3 < 1 || p1 > 60 || p2 > 60 || p3 > 60) return -1;
    memset(G, 0, sizeof(double) * (size_t)N * N);
    if (path == ORC_GENERAL) {
        if (L < 1 || L > 32) return -1;
        double *wg = NULL;
        const double *w = wgrid;
        if (!w) {
            wg = malloc(sizeof(double) * L * L * L);
            for (int t = 0; t < L * L * L; ++t) wg[t] = coef;
            w = wg;
        }
        long long acc = -1;
        switch (space) {
        case ORC_L2: acc = tens_l2(p1, p2, p3, L, nodes, weights, kind, par, w, G); break;
        case ORC_H1: acc = tens_h1(p1, p2, p3, L, nodes, weights, kind, par, w, G); break;
        case ORC_HDIV: acc = tens_hdiv(p1, p2, p3, L, nodes, weights, kind, par, w, G); break;
        case ORC_HCURL: acc = tens_hcurl(p1, p2, p3, L, nodes, weights, kind, par, w, G); break;
        }
        free(wg);
        return acc;
    }
    if (path == ORC_EXTRUSION ? kind > 3 : kind > 2) return -1; /* gram.py:170-174 */
    int pm = p1 > p2 ? p1 : p2;
    pm = pm > p3 ? pm : p3;
    int pF = pm + 1 > 2 ? pm + 1 : 2; /* gram.py:228-231 */
    int nF = pF + 1;
    double *fall = malloc(sizeof(double) * 4 * nF * nF);
    orc_ftable(pF, fall);
    long long acc = -1;
    if (path == ORC_EXTRUSION) { /* gram.py:192-203: rule in (xi2, xi3), F tables in xi1 */
        if (L < 1 || L > 32 || !nodes || !weights) { free(fall); return -1; }
        switch (space) {
        case ORC_L2: acc = simp_l2_ext(p1, p2, p3, fall, nF, L, nodes, weights, kind, par, coef, G); break;
        case ORC_H1: acc = simp_h1_ext(p1, p2, p3, fall, nF, L, nodes, weights, kind, par, coef, G); break;
        case ORC_HDIV: acc = simp_hdiv_ext(p1, p2, p3, fall, nF, L, nodes, weights, kind, par, coef, G); break;
        case ORC_HCURL: acc = simp_hcurl_ext(p1, p2, p3, fall, nF, L, nodes, weights, kind, par, coef, G); break;
        }
        free(fall);
        return acc;
    }
    switch (space) {
    case ORC_L2: acc = simp_l2(p1, p2, p3, fall, nF, kind, par, coef, G); break;
    case ORC_H1: acc = simp_h1(p1, p2, p3, fall, nF, kind, par, coef, G); break;
    case ORC_HDIV: acc = simp_hdiv(p1, p2, p3, fall, nF, kind, par, coef, G); break;
    case ORC_HCURL: acc = simp_hcurl(p1, p2, p3, fall, nF, kind, par, coef, G); break;
    }
    free(fall);
    return acc;
}

/* Batched: E independent elements, packed upper triangles out[E][N(N+1)/2].
 * A pthread pool pulls elements from an atomic counter (the reference
 * kernels are serial and hold the GIL; SPEC.md:380-381 states that every
 * gram_* call is pure and independent, so elements run concurrently). */
typedef struct {
    int space, path, p1, p2, p3, L, E, N;
    const int *kind;
    const double *params, *coef, *wgrid;
    double *out;
    const double *nodes, *weights;
    int next;
    int bad;
} orc_job;

static void *orc_worker(void *arg)
{
    orc_job *j = (orc_job *)arg;
    size_t P = (size_t)j->N * (j->N + 1) / 2;
    double *G = malloc(sizeof(double) * (size_t)j->N * j->N);
    for (;;) {
        int e = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (e >= j->E) break;
        const double *wg = j->wgrid ? j->wgrid + (size_t)e * j->L * j->L * j->L : NULL;
        long long acc = orc_gram_full(j->space, j->path, j->p1, j->p2, j->p3, j->L, j->nodes,
                                      j->weights, j->kind[e], j->params + (size_t)24 * e,
                                      j->coef ? j->coef[e] : 1.0, wg, G);
        if (acc < 0) { __atomic_store_n(&j->bad, 1, __ATOMIC_RELAXED); continue; }
        double *o = j->out + P * e;
        size_t k = 0;
        for (int r = 0; r < j->N; ++r)
            for (int c = r; c < j->N; ++c) o[k++] = G[(size_t)r * j->N + c];
    }
    free(G);
    return NULL;
}

int orc_num_cpus(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

int orc_gram_batched(int space, int path, int p1, int p2, int p3, int L, int E,
                     const int *kind, const double *params, const double *coef,
                     const double *wgrid, double *out, int nthreads)
{
    int N = orc_dim(space, p1, p2, p3);
    if (N <= 0 || E < 0) return -1;
    double nodes[32], weights[32];
    if (path != ORC_AFFINE && orc_gauss_rule(L, nodes, weights) != 0) return -1;
    orc_job job = {space, path, p1, p2, p3, L, E, N, kind, params, coef, wgrid, out,
                   nodes, weights, 0, 0};
    if (nthreads <= 0) nthreads = orc_num_cpus();
    if (nthreads > 256) nthreads = 256;
    if (nthreads == 1) {
        orc_worker(&job);
    } else {
        pthread_t th[256];
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, orc_worker, &job);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    return job.bad ? -1 : 0;
}
