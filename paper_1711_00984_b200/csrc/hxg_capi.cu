// hxg_capi.cu -- host side of libhexgram_b200.so: space planner, launch
// configuration and the extern "C" entry points declared in
// include/hexgram_b200.h.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/hexgram_b200.h"
#include "hxg_affine_v2.cuh"
#include "hxg_extrusion.cuh"
#include "hxg_general_v2.cuh"
#include "hxg_device.h"
#include "hxg_kernels.cuh"
#include "hxg_v2_launch.h"
#include <cstdlib>

using namespace hxg;

namespace {

// ---------------------------------------------------------------------------
// planner: blocks, terms and stage groups per space (see hxg_plan.h)
// ---------------------------------------------------------------------------
struct HostTerm {
    int field, sign, r[3], s[3];
};

int build_plan(int space, int p1, int p2, int p3, SpacePlan &P)
{
    const int p[3] = {p1, p2, p3};
    for (int d = 0; d < 3; ++d)
        if (p[d] < 1 || p[d] > HXG_MAX_ORDER) return HXG_ERR_ORDER;
    memset(&P, 0, sizeof(P));
    P.space = space;
    int prim[3][3] = {{0}};  // function code of the r = 0 factor: 0 chi, 1 chi'
    switch (space) {
    case H1:  // spaces.py:67-72, phi = chi chi chi
        P.nb = 1;
        P.nfields = 7;
        for (int d = 0; d < 3; ++d) { P.n[0][d] = p[d] + 1; P.sh[0][d] = 0; prim[0][d] = 0; }
        break;
    case L2:  // nu_i = chi'_{i+1}  (poly1d.py:1-13)
        P.nb = 1;
        P.nfields = 1;
        for (int d = 0; d < 3; ++d) { P.n[0][d] = p[d]; P.sh[0][d] = 1; prim[0][d] = 1; }
        break;
    case HDIV:  // spaces.py:95-102, shape3_eval 201-213: chi on a, nu elsewhere
        P.nb = 3;
        P.nfields = 7;
        for (int a = 0; a < 3; ++a)
            for (int d = 0; d < 3; ++d) {
                P.n[a][d] = d == a ? p[d] + 1 : p[d];
                P.sh[a][d] = d == a ? 0 : 1;
                prim[a][d] = d == a ? 0 : 1;
            }
        break;
    case HCURL:  // spaces.py:95-102, shape3_eval 215-232: nu on a, chi elsewhere
        P.nb = 3;
        P.nfields = 12;
        for (int a = 0; a < 3; ++a)
            for (int d = 0; d < 3; ++d) {
                P.n[a][d] = d == a ? p[d] : p[d] + 1;
                P.sh[a][d] = d == a ? 1 : 0;
                prim[a][d] = d == a ? 1 : 0;
            }
        break;
    default:
        return HXG_ERR_SPACE;
    }
    int off = 0;
    for (int a = 0; a < P.nb; ++a) {
        P.off[a] = off;
        off += P.n[a][0] * P.n[a][1] * P.n[a][2];
    }
    P.N = off;
    for (int a = 0; a < P.nb; ++a)
        for (int b = 0; b < P.nb; ++b) {
            std::vector<HostTerm> terms;
            auto unit = [](int d, int k) { return d == k ? 1 : 0; };
            if (space == H1) {
                terms.push_back({0, 1, {0, 0, 0}, {0, 0, 0}});
                for (int al = 0; al < 3; ++al)
                    for (int be = 0; be < 3; ++be)
                        terms.push_back({1 + sym3(al, be), 1,
                                         {unit(0, al), unit(1, al), unit(2, al)},
                                         {unit(0, be), unit(1, be), unit(2, be)}});
            } else if (space == L2) {
                terms.push_back({0, 1, {0, 0, 0}, {0, 0, 0}});
            } else if (space == HDIV) {
                terms.push_back({sym3(a, b), 1, {0, 0, 0}, {0, 0, 0}});
                terms.push_back({6, 1, {unit(0, a), unit(1, a), unit(2, a)},
                                 {unit(0, b), unit(1, b), unit(2, b)}});
            } else {  // HCURL: curl comp a+1 = +..., comp a+2 = -... (spaces.py:222-231)
                terms.push_back({sym3(a, b), 1, {0, 0, 0}, {0, 0, 0}});
                for (int al = 0; al < 2; ++al)
                    for (int be = 0; be < 2; ++be) {
                        const int ca = (a + al + 1) % 3, cb = (b + be + 1) % 3;
                        HostTerm t;
                        t.field = 6 + sym3(ca, cb);
                        t.sign = al == be ? 1 : -1;
                        for (int d = 0; d < 3; ++d) {
                            t.r[d] = (d != a && d != ca) ? 1 : 0;
                            t.s[d] = (d != b && d != cb) ? 1 : 0;
                        }
                        terms.push_back(t);
                    }
            }
            // resolve function codes and group: g by (f0, f1) pairs, h by f0 pair
            PairPlan &pp = P.pair[a][b];
            std::vector<int> gkeys, hkeys;
            struct R { int field, sign, fr[3], fs[3]; };
            std::vector<R> rt;
            for (auto &t : terms) {
                R r;
                r.field = t.field;
                r.sign = t.sign;
                for (int d = 0; d < 3; ++d) {
                    r.fr[d] = t.r[d] ? 1 : prim[a][d];
                    r.fs[d] = t.s[d] ? 1 : prim[b][d];
                }
                rt.push_back(r);
            }
            // order terms by g so that stage A iterates groups contiguously
            std::vector<int> tg(rt.size());
            for (size_t i = 0; i < rt.size(); ++i) {
                const int gk = ((rt[i].fr[0] * 2 + rt[i].fs[0]) * 2 + rt[i].fr[1]) * 2 + rt[i].fs[1];
                auto it = std::find(gkeys.begin(), gkeys.end(), gk);
                if (it == gkeys.end()) { gkeys.push_back(gk); tg[i] = (int)gkeys.size() - 1; }
                else tg[i] = (int)(it - gkeys.begin());
            }
            pp.ng = (int8_t)gkeys.size();
            for (size_t g = 0; g < gkeys.size(); ++g) {
                const int gk = gkeys[g];
                const int hk = gk >> 2;
                auto it = std::find(hkeys.begin(), hkeys.end(), hk);
                int h;
                if (it == hkeys.end()) { hkeys.push_back(hk); h = (int)hkeys.size() - 1; }
                else h = (int)(it - hkeys.begin());
                pp.g_h[g] = (int8_t)h;
                pp.g_fr[g] = (int8_t)((gk >> 1) & 1);
                pp.g_fs[g] = (int8_t)(gk & 1);
            }
            pp.nh = (int8_t)hkeys.size();
            for (size_t h = 0; h < hkeys.size(); ++h) {
                pp.h_fr[h] = (int8_t)((hkeys[h] >> 1) & 1);
                pp.h_fs[h] = (int8_t)(hkeys[h] & 1);
            }
            int nt = 0;
            for (int g = 0; g < pp.ng; ++g)
                for (size_t i = 0; i < rt.size(); ++i)
                    if (tg[i] == g) {
                        pp.t_g[nt] = (int8_t)g;
                        pp.t_field[nt] = (int8_t)rt[i].field;
                        pp.t_fr[nt] = (int8_t)rt[i].fr[2];
                        pp.t_fs[nt] = (int8_t)rt[i].fs[2];
                        pp.t_sign[nt] = (int8_t)rt[i].sign;
                        ++nt;
                    }
            pp.nt = (int8_t)nt;
        }
    return HXG_OK;
}

// ---------------------------------------------------------------------------
// launch configuration of the general kernel
// ---------------------------------------------------------------------------
constexpr size_t GEN_SMEM_BUDGET = 110 * 1024;  // two CTAs per SM (228 KB per SM)
constexpr size_t GEN_SMEM_MAX = 220 * 1024;

struct GenConfig {
    int R2, R3, N2, NG, NH, SLD, LP;
    int off_T, off_A, off_B, off_S;
    size_t smem;
};

GenConfig gen_config(const SpacePlan &P, int L, size_t budget)
{
    GenConfig c{};
    c.LP = (L + 1) & ~1;
    int n1max = 0, n2max = 0, n3max = 0, c12max = 0;
    c.NG = 1;
    c.NH = 1;
    for (int a = 0; a < P.nb; ++a) {
        n1max = std::max(n1max, P.n[a][0]);
        n2max = std::max(n2max, P.n[a][1]);
        n3max = std::max(n3max, P.n[a][2]);
        c12max = std::max(c12max, P.n[a][0] * P.n[a][1]);
        for (int b = 0; b < P.nb; ++b) {
            c.NG = std::max(c.NG, (int)P.pair[a][b].ng);
            c.NH = std::max(c.NH, (int)P.pair[a][b].nh);
        }
    }
    c.N2 = n2max;
    auto sizes = [&](int R2, int R3, GenConfig &g) {
        g.R2 = R2;
        g.R3 = R3;
        g.SLD = ((c12max * R3 + 7) / 8) * 8 + 2;  // +2 doubles: spread banks across rows
        g.off_T = 0;
        g.off_A = g.off_T + 2 * KT * c.LP;
        g.off_B = g.off_A + R3 * c.NG * L * c.LP;
        g.off_S = g.off_B + R2 * c.NH * R3 * c.N2 * c.LP;
        const int total = g.off_S + R2 * n1max * g.SLD;
        g.smem = (size_t)total * sizeof(double);
    };
    GenConfig best = c;
    bool found = false;
    for (int R3 = n3max; R3 >= 1 && !found; --R3) {
        GenConfig g = c;
        sizes(n2max, R3, g);
        if (g.smem <= budget) { best = g; found = true; }
    }
    for (int R2 = n2max; R2 >= 1 && !found; --R2) {
        GenConfig g = c;
        sizes(R2, 1, g);
        if (g.smem <= budget) { best = g; found = true; }
    }
    if (!found) sizes(1, 1, best);
    return best;
}

template <int LMAX, int NMT>
int launch_general_t(const GenArgs &args, size_t smem, int grid, cudaStream_t st)
{
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(general_kernel<LMAX, NMT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)GEN_SMEM_MAX);
    });
    if (attr_err != cudaSuccess) return HXG_ERR_CUDA;
    general_kernel<LMAX, NMT><<<grid, GEN_THREADS, smem, st>>>(args);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

int launch_affine(const AffArgs &args, size_t smem, int grid, cudaStream_t st)
{
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(affine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(64 * 1024));
    });
    if (attr_err != cudaSuccess) return HXG_ERR_CUDA;
    affine_kernel<<<grid, AFF_THREADS, smem, st>>>(args);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

size_t metric_bytes_per_element(const SpacePlan &P, int L)
{
    return (size_t)P.nfields * L * L * L * sizeof(double);
}

constexpr size_t WS_TARGET = 512ull << 20;  // metric workspace per launch chunk

int elements_per_chunk(const SpacePlan &P, int L, int E, size_t ws_bytes)
{
    const size_t per = metric_bytes_per_element(P, L);
    size_t cap = ws_bytes / per;
    if (cap > (size_t)E) cap = E;
    if (cap > (1u << 24)) cap = 1u << 24;
    return (int)cap;
}

int check_common(int space, int path, int p1, int p2, int p3, int L, int E)
{
    if (space < 0 || space > 3 || path < 0 || path > 2) return HXG_ERR_SPACE;
    if (p1 < 1 || p2 < 1 || p3 < 1 || p1 > HXG_MAX_ORDER || p2 > HXG_MAX_ORDER || p3 > HXG_MAX_ORDER)
        return HXG_ERR_ORDER;
    if (path != AFFINE && (L < 1 || L > HXG_MAX_RULE)) return HXG_ERR_ORDER;
    if (E < 0) return HXG_ERR_ARG;
    return HXG_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// extrusion path, anisotropic orders with a rule too short for xi1 (L < p1 + 1):
// the reference integrates xi1 exactly (F tables) and (xi2, xi3) with the L-point
// rule.  The hierarchical bases are nested, so the anisotropic Gram is the
// sub-matrix of the isotropic order-p = max(p_d) Gram (computed by the exact
// extrusion kernel with the same rule) on the basis functions the orders keep.
// ---------------------------------------------------------------------------
__device__ int ext_iso_index(int space, int r, int p1, int p2, int p3, int p)
{
    const int pd[3] = {p1, p2, p3};
    if (space == H1 || space == L2) {
        const int s = space == H1 ? 1 : 0;
        const int q0 = pd[0] + s, q1 = pd[1] + s, Q = p + s;
        const int i1 = r % q0, i2 = (r / q0) % q1, i3 = r / (q0 * q1);
        return i1 + Q * (i2 + Q * i3);
    }
    int off = 0, offI = 0;
    for (int a = 0; a < 3; ++a) {
        int n[3], Nn[3];
        for (int d = 0; d < 3; ++d) {
            const int e = space == HDIV ? (d == a) : (d != a);
            n[d] = pd[d] + e;
            Nn[d] = p + e;
        }
        const int sz = n[0] * n[1] * n[2];
        if (r < off + sz) {
            const int x = r - off;
            const int i1 = x % n[0], i2 = (x / n[0]) % n[1], i3 = x / (n[0] * n[1]);
            return offI + i1 + Nn[0] * (i2 + Nn[1] * i3);
        }
        off += sz;
        offI += Nn[0] * Nn[1] * Nn[2];
    }
    return -1;
}

__global__ void ext_gather_kernel(int space, int p1, int p2, int p3, int p, int N, int Niso, int E,
                                  const double *__restrict__ iso, double *__restrict__ out)
{
    const long long P = (long long)N * (N + 1) / 2, Piso = (long long)Niso * (Niso + 1) / 2;
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long row = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); row < (long long)E * N;
         row += nw) {
        const long long e = row / N;
        const int r = (int)(row - e * N);
        const int R = ext_iso_index(space, r, p1, p2, p3, p);
        const double *src = iso + e * Piso + (long long)R * Niso - (long long)R * (R - 1) / 2 - R;
        double *dst = out + e * P + (long long)r * N - (long long)r * (r - 1) / 2 - r;
        for (int c = r + lane; c < N; c += 32) dst[c] = src[ext_iso_index(space, c, p1, p2, p3, p)];
    }
}

static bool ext_gather_route(int path, int p1, int p2, int p3, int L)
{
    return path == EXTRUSION && !(p1 == p2 && p2 == p3) && L < p1 + 1;
}

// the specialized metric kernel covers L = 2..11 and writes every status word itself
static bool metric_v2_ok(int space, int L)
{
    const char *fg = getenv("HXG_FORCE_GENERIC");
    return space >= 0 && space <= 3 && L >= 2 && L <= 11 && !(fg && fg[0] == '1');
}

static int metric_run(int space, int p1, int p2, int p3, int L, int E, const int *kind,
                       const double *params, const double *coef, const double *wgrid,
                       const double *tables, double *metric, int *status, void *stream,
                       bool status_whole)
{
    int rc = check_common(space, GENERAL, p1, p2, p3, L, E);
    if (rc != HXG_OK) return rc;
    if (E == 0) return HXG_OK;
    if (!kind || !params || !tables || !metric || !status) return HXG_ERR_ARG;
    SpacePlan P;
    rc = build_plan(space, p1, p2, p3, P);
    if (rc != HXG_OK) return rc;
    // compile-time specialized kernel (writes whole status words) unless the generic one is forced
    const char *fg = getenv("HXG_FORCE_GENERIC");
    if (metric_v2_ok(space, L) && !(fg && fg[0] == '1')) {
        MetArgs a{E, kind, params, coef, wgrid, tables, metric, status, status_whole ? 0 : 1};
        int r = 1;
        switch (space) {
        case H1: r = launch_met_H1(L, a, (cudaStream_t)stream); break;
        case HCURL: r = launch_met_hcurl(L, a, (cudaStream_t)stream); break;
        case HDIV: r = launch_met_hdiv(L, a, (cudaStream_t)stream); break;
        case L2: r = launch_met_l2(L, a, (cudaStream_t)stream); break;
        }
        if (r <= 0) return r == 0 ? HXG_OK : HXG_ERR_CUDA;
    }
    const long long npts = (long long)E * L * L * L;
    const int mgrid = (int)std::min<long long>((npts + 255) / 256, (long long)sm_count() * 64);
    metric_kernel<<<mgrid, 256, 0, (cudaStream_t)stream>>>(space, L, E, kind, params, coef, wgrid,
                                                         tables, metric, status, P.nfields);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

// ===========================================================================
// extern "C" API
// ===========================================================================
extern "C" {

int hxg_version(void) { return 100; }

int hxg_fused_order_max(void) { return hxg::fused_order_max(); }

const char *hxg_error_string(int code)
{
    switch (code) {
    case HXG_OK: return "ok";
    case HXG_ERR_ORDER: return "order or rule size outside the supported range";
    case HXG_ERR_SPACE: return "unknown space or path";
    case HXG_ERR_KIND: return "map kind admits no simplification (constant-Jacobian path needs kind <= 2)";
    case HXG_ERR_WORKSPACE: return "workspace too small";
    case HXG_ERR_CUDA: return "CUDA error";
    case HXG_ERR_ARG: return "invalid argument";
    case HXG_ERR_DEGENERATE: return "element map with det J <= 0 at a quadrature point";
    }
    return "unknown error";
}

int hxg_dim(int space, int p1, int p2, int p3)
{
    SpacePlan P;
    const int rc = build_plan(space, p1, p2, p3, P);
    return rc == HXG_OK ? P.N : rc;
}

long long hxg_accumulations(int space, int path, int p1, int p2, int p3, int L)
{
    // closed forms of OpCounters.accumulations (verified against
    // the reference kernels: tensorized T L N(N+1)/2, simplified T N(N+1)/2,
    // L2 L (p(p+1)/2)^3 with per-direction products for anisotropic orders)
    const int N = hxg_dim(space, p1, p2, p3);
    if (N < 0) return N;
    if (space == L2) {
        const long long t = (long long)p1 * (p1 + 1) / 2 * ((long long)p2 * (p2 + 1) / 2) *
                            ((long long)p3 * (p3 + 1) / 2);
        return path == GENERAL ? L * t : t;
    }
    const long long T = space == H1 ? 10 : (space == HCURL ? 5 : 2);
    const long long tri = (long long)N * (N + 1) / 2;
    return path == GENERAL ? T * L * tri : T * tri;
}

size_t hxg_tables_doubles(void) { return TAB_TOTAL; }

int hxg_make_tables(int L, const double *nodes, const double *weights, double *tables, void *stream)
{
    if (L < 1 || L > LT) return HXG_ERR_ORDER;
    if (!tables) return HXG_ERR_ARG;
    if ((nodes == nullptr) != (weights == nullptr)) return HXG_ERR_ARG;
    tables_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(L, nodes, weights, tables);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

size_t hxg_workspace_size(int space, int path, int p1, int p2, int p3, int L, int E)
{
    if (check_common(space, path, p1, p2, p3, L, E) != HXG_OK) return 0;
    if (path == AFFINE || E == 0) return 0;
    if (ext_gather_route(path, p1, p2, p3, L)) {  // isotropic order-max(p) Grams per chunk
        const int p = std::max(p1, std::max(p2, p3));
        if (p > 10) return 0;
        const size_t per = sizeof(double) * (size_t)hxg_dim(space, p, p, p) * (hxg_dim(space, p, p, p) + 1) / 2;
        return std::min<size_t>((size_t)E, std::max<size_t>(1, WS_TARGET / per)) * per;
    }
    if (path == EXTRUSION && p1 == p2 && p2 == p3 && p1 <= 10 &&
        !(getenv("HXG_FORCE_GENERIC") && getenv("HXG_FORCE_GENERIC")[0] == '1'))
        return 0;  // specialized kernel, no metric workspace
    SpacePlan P;
    build_plan(space, p1, p2, p3, P);
    const size_t per = metric_bytes_per_element(P, L);
    size_t n = (size_t)E;
    const size_t cap = std::max<size_t>(1, WS_TARGET / per);
    if (n > cap) n = cap;
    return n * per;
}

int hxg_gram_batched(int space, int path, int p1, int p2, int p3, int L, int E, const int *kind,
                     const double *params, const double *coef, const double *wgrid,
                     const double *tables, double *out, int *status, void *workspace,
                     size_t workspace_bytes, void *stream)
{
    int rc = check_common(space, path, p1, p2, p3, L, E);
    if (rc != HXG_OK) return rc;
    if (E == 0) return HXG_OK;
    if (!kind || !params || !tables || !out || !status) return HXG_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    SpacePlan P;
    rc = build_plan(space, p1, p2, p3, P);
    if (rc != HXG_OK) return rc;
    const long long Pk = (long long)P.N * (P.N + 1) / 2;
    // every kernel but the specialized affine one ORs flags into a zeroed status word
    const char *force_generic = getenv("HXG_FORCE_GENERIC");
    const bool aff_spec = path == AFFINE && p1 == p2 && p2 == p3 && p1 <= 10 &&
                          !(force_generic && force_generic[0] == '1');
    // general path, unfused orders: the specialized metric kernel writes the words whole
    const char *force_v2 = getenv("HXG_FORCE_V2");
    const bool fused_gen = path == GENERAL && p1 == p2 && p2 == p3 && p1 <= fused_order_max() && L == p1 + 1 &&
                           !(force_generic && force_generic[0] == '1') && !(force_v2 && force_v2[0] == '1');
    const bool met_writes = path == GENERAL && !fused_gen && metric_v2_ok(space, L) &&
                            !ext_gather_route(path, p1, p2, p3, L);
    if (!aff_spec && !met_writes && cudaMemsetAsync(status, 0, sizeof(int) * (size_t)E, st) != cudaSuccess)
        return HXG_ERR_CUDA;

    if (path == AFFINE) {
        const char *force = force_generic;
        if (p1 == p2 && p2 == p3 && !(force && force[0] == '1')) {
            // compile-time specialized kernel (isotropic p <= 10), chunked below 2^31 blocks
            const long long units = P.nb == 1 ? (long long)P.n[0][1] * P.n[0][2]
                                              : (long long)P.n[0][1] * P.n[0][2] + P.n[1][1] * P.n[1][2] +
                                                    P.n[2][1] * P.n[2][2];
            const long long maxE = std::max<long long>(1, ((1ll << 31) - 1) / units);
            int r = 0;
            for (long long e0 = 0; e0 < E && r == 0; e0 += maxE) {
                AffV2Args a2;
                a2.kind = kind + e0;
                a2.params = params + 24 * e0;
                a2.coef = coef ? coef + e0 : nullptr;
                a2.tables = tables;
                a2.out = out + e0 * Pk;
                a2.status = status + e0;
                a2.P = Pk;
                a2.E = (int)std::min<long long>(maxE, E - e0);
                switch (space) {
                case H1: r = launch_aff_H1(p1, a2, st); break;
                case HCURL: r = launch_aff_hcurl(p1, a2, st); break;
                case HDIV: r = launch_aff_hdiv(p1, a2, st); break;
                default: r = launch_aff_l2(p1, a2, st); break;
                }
            }
            if (r <= 0) return r == 0 ? HXG_OK : HXG_ERR_CUDA;
            if (aff_spec && cudaMemsetAsync(status, 0, sizeof(int) * (size_t)E, st) != cudaSuccess)
                return HXG_ERR_CUDA;  // no specialization after all: the generic kernel ORs flags
        }
        AffArgs a;
        memset(&a, 0, sizeof(a));
        a.plan = P;
        a.E = E;
        int tot = 0, n2 = 0, n3 = 0;
        for (int b = 0; b < P.nb; ++b) {
            a.ucount[b] = P.n[b][1] * P.n[b][2];
            tot += a.ucount[b];
            n2 = std::max(n2, P.n[b][1]);
            n3 = std::max(n3, P.n[b][2]);
        }
        a.nunits_total = tot;
        a.N2 = n2;
        a.N3 = n3;
        a.kind = kind;
        a.params = params;
        a.coef = coef;
        a.tables = tables;
        a.status = status;
        a.P = Pk;
        const size_t smem = (size_t)(4 * KT * KT + 3 * n3 * n2 * MAXH) * sizeof(double);
        // kind check (gram.py:170-174): the host layer validates kinds before the
        // call; grids are chunked to stay below 2^31 blocks
        const long long maxE = std::max<long long>(1, (1ll << 31) / std::max(tot, 1) - 1);
        for (long long e0 = 0; e0 < E; e0 += maxE) {
            const int ne = (int)std::min<long long>(maxE, E - e0);
            AffArgs c = a;
            c.E = ne;
            c.kind = kind + e0;
            c.params = params + 24 * e0;
            c.coef = coef ? coef + e0 : nullptr;
            c.status = status + e0;
            c.out = out + e0 * Pk;
            rc = launch_affine(c, smem, ne * tot, st);
            if (rc != HXG_OK) return rc;
        }
        return HXG_OK;
    }

    if (path == EXTRUSION) {
        // simplified extrusion path (simp_*_ext): compile-time specialized kernel for
        // isotropic p <= 10; otherwise the general kernels with the same rule compute
        // the same integral (the xi1 quadrature with L = p + 1 points is exact for an
        // xi1-independent Jacobian), after the kind check of gram.py:170-174
        const char *force = getenv("HXG_FORCE_GENERIC");
        if (p1 == p2 && p2 == p3 && !(force && force[0] == '1')) {
            ExtArgs x;
            x.kind = kind;
            x.params = params;
            x.coef = coef;
            x.tables = tables;
            x.out = out;
            x.status = status;
            x.P = Pk;
            x.E = E;
            x.rg = 1;
            x.L = L;
            x.jc = 1;
            int r = 1;
            switch (space) {
            case H1: r = launch_ext_H1(p1, x, st); break;
            case HCURL: r = launch_ext_hcurl(p1, x, st); break;
            case HDIV: r = launch_ext_hdiv(p1, x, st); break;
            default: r = launch_ext_l2(p1, x, st); break;
            }
            if (r <= 0) return r == 0 ? HXG_OK : HXG_ERR_CUDA;
        }
        if (ext_gather_route(path, p1, p2, p3, L)) {
            const int p = std::max(p1, std::max(p2, p3));
            if (p > 10) return HXG_ERR_ORDER;  // no exact-xi1 kernel above p = 10
            const int N = hxg_dim(space, p1, p2, p3), Ni = hxg_dim(space, p, p, p);
            const size_t per = sizeof(double) * (size_t)Ni * (Ni + 1) / 2;
            if (!workspace || workspace_bytes < per) return HXG_ERR_WORKSPACE;
            const int chunk = (int)std::min<size_t>((size_t)E, workspace_bytes / per);
            for (int e0 = 0; e0 < E; e0 += chunk) {
                const int ne = std::min(chunk, E - e0);
                ExtArgs x;
                x.kind = kind + e0;
                x.params = params + 24LL * e0;
                x.coef = coef ? coef + e0 : nullptr;
                x.tables = tables;
                x.out = (double *)workspace;
                x.status = status + e0;
                x.P = (long long)Ni * (Ni + 1) / 2;
                x.E = ne;
                x.rg = 1;
                x.L = L;
                x.jc = 1;
                int r = 1;
                switch (space) {
                case H1: r = launch_ext_H1(p, x, st); break;
                case HCURL: r = launch_ext_hcurl(p, x, st); break;
                case HDIV: r = launch_ext_hdiv(p, x, st); break;
                default: r = launch_ext_l2(p, x, st); break;
                }
                if (r != 0) return HXG_ERR_CUDA;
                const long long rows = (long long)ne * N;
                ext_gather_kernel<<<(int)std::min<long long>((rows + 7) / 8, (long long)sm_count() * 64), 256, 0, st>>>(
                    space, p1, p2, p3, p, N, Ni, ne, (const double *)workspace, out + (long long)e0 * Pk);
                if (cudaGetLastError() != cudaSuccess) return HXG_ERR_CUDA;
            }
            return HXG_OK;
        }
        ext_kind_kernel<<<(E + 255) / 256, 256, 0, st>>>(E, kind, status);
        if (cudaGetLastError() != cudaSuccess) return HXG_ERR_CUDA;
    }

    // general path, low isotropic orders: one fused kernel (geometry evaluated in
    // the contraction kernel, no metric pass / workspace)
    {
        const char *fg = getenv("HXG_FORCE_GENERIC"), *f2 = getenv("HXG_FORCE_V2");
        if (p1 == p2 && p2 == p3 && p1 <= fused_order_max() && L == p1 + 1 && !(fg && fg[0] == '1') &&
            !(f2 && f2[0] == '1')) {
            V2Args a;
            a.tables = tables;
            a.metric = nullptr;
            a.out = out;
            a.P = Pk;
            a.E = E;
            a.kind = kind;
            a.params = params;
            a.coef = coef;
            a.wgrid = wgrid;
            a.status = status;
            int r = 1;
            switch (space) {
            case H1: r = launch_v2_H1(p1, a, st); break;
            case HCURL: r = launch_v2_hcurl(p1, a, st); break;
            case HDIV: r = launch_v2_hdiv(p1, a, st); break;
            case L2: r = launch_v2_l2(p1, a, st); break;
            }
            if (r <= 0) return r == 0 ? HXG_OK : HXG_ERR_CUDA;
        }
    }
    // general path: metric kernel then the three-stage contraction, per chunk
    if (!workspace) return HXG_ERR_WORKSPACE;
    const int Ech = elements_per_chunk(P, L, E, workspace_bytes);
    if (Ech < 1) return HXG_ERR_WORKSPACE;
    for (long long e0 = 0; e0 < E; e0 += Ech) {
        const int ne = (int)std::min<long long>(Ech, E - e0);
        double *metric = (double *)workspace;
        rc = metric_run(space, p1, p2, p3, L, ne, kind + e0, params + 24 * e0,
                                coef ? coef + e0 : nullptr, wgrid ? wgrid + e0 * L * L * L : nullptr,
                                tables, metric, status + e0, stream, met_writes);
        if (rc != HXG_OK) return rc;
        rc = hxg_contract_batched(space, p1, p2, p3, L, ne, tables, metric, out + e0 * Pk, stream);
        if (rc != HXG_OK) return rc;
    }
    return HXG_OK;
}

int hxg_metric_batched(int space, int p1, int p2, int p3, int L, int E, const int *kind,
                       const double *params, const double *coef, const double *wgrid,
                       const double *tables, double *metric, int *status, void *stream)
{
    // exported entry: the status word is written by the call (zeroed, then ORed; the
    // specialized metric kernel writes it whole)
    if (E > 0 && status && !metric_v2_ok(space, L) && cudaMemsetAsync(status, 0, sizeof(int) * (size_t)E, (cudaStream_t)stream) != cudaSuccess)
        return HXG_ERR_CUDA;
    return metric_run(space, p1, p2, p3, L, E, kind, params, coef, wgrid, tables, metric, status, stream, true);
}

int hxg_contract_batched(int space, int p1, int p2, int p3, int L, int E, const double *tables,
                         const double *metric, double *out, void *stream)
{
    int rc = check_common(space, GENERAL, p1, p2, p3, L, E);
    if (rc != HXG_OK) return rc;
    if (E == 0) return HXG_OK;
    if (!tables || !metric || !out) return HXG_ERR_ARG;
    SpacePlan P;
    rc = build_plan(space, p1, p2, p3, P);
    if (rc != HXG_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    // compile-time specialized kernels: isotropic p <= 10 with L = p + 1
    // (HXG_FORCE_GENERIC=1 selects the runtime-generic kernel, for testing)
    const char *force = getenv("HXG_FORCE_GENERIC");
    if (p1 == p2 && p2 == p3 && L == p1 + 1 && !(force && force[0] == '1')) {
        V2Args a;
        a.tables = tables;
        a.metric = metric;
        a.out = out;
        a.P = (long long)P.N * (P.N + 1) / 2;
        a.E = E;
        int r = 1;
        switch (space) {
        case H1: r = launch_v2_H1(p1, a, st); break;
        case HCURL: r = launch_v2_hcurl(p1, a, st); break;
        case HDIV: r = launch_v2_hdiv(p1, a, st); break;
        case L2: r = launch_v2_l2(p1, a, st); break;
        }
        if (r <= 0) return r == 0 ? HXG_OK : HXG_ERR_CUDA;
    }
    GenArgs g;
    memset(&g, 0, sizeof(g));
    g.plan = P;
    g.L = L;
    g.E = E;
    const GenConfig cfg = gen_config(P, L, GEN_SMEM_BUDGET);
    if (cfg.smem > GEN_SMEM_MAX) return HXG_ERR_ORDER;
    g.LP = cfg.LP;
    g.R2 = cfg.R2;
    g.R3 = cfg.R3;
    g.N2 = cfg.N2;
    g.NG = cfg.NG;
    g.NH = cfg.NH;
    g.SLD = cfg.SLD;
    g.off_T = cfg.off_T;
    g.off_A = cfg.off_A;
    g.off_B = cfg.off_B;
    g.off_S = cfg.off_S;
    g.tables = tables;
    g.metric = metric;
    g.out = out;
    g.P = (long long)P.N * (P.N + 1) / 2;
    int nu = 0;
    for (int b = 0; b < P.nb; ++b)
        for (int j3 = 0; j3 < P.n[b][2]; ++j3) {
            g.unit_b[nu] = (int8_t)b;
            g.unit_j3[nu] = (int8_t)j3;
            ++nu;
        }
    g.nunits = nu;
    int n1max = 0;
    for (int a = 0; a < P.nb; ++a) n1max = std::max(n1max, P.n[a][0]);
    const int nmt = n1max <= 8 ? 1 : 2;
    const long long grid = (long long)E * nu;
    if (grid >= (1ll << 31)) return HXG_ERR_ARG;
    if (L <= 8) rc = nmt == 1 ? launch_general_t<8, 1>(g, cfg.smem, (int)grid, st)
                              : launch_general_t<8, 2>(g, cfg.smem, (int)grid, st);
    else rc = nmt == 1 ? launch_general_t<16, 1>(g, cfg.smem, (int)grid, st)
                       : launch_general_t<16, 2>(g, cfg.smem, (int)grid, st);
    return rc;
}

int hxg_expand_full(int N, int E, const double *packed, double *full, void *stream)
{
    if (N < 1 || E < 0 || !packed || !full) return HXG_ERR_ARG;
    const long long total = (long long)E * N * N;
    if (total == 0) return HXG_OK;
    const int grid = (int)std::min<long long>((total + 255) / 256, (long long)sm_count() * 32);
    expand_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(N, total, packed, full);
    return cudaGetLastError() == cudaSuccess ? HXG_OK : HXG_ERR_CUDA;
}

// Host-buffer entry: the reference's calling convention (numpy in, numpy out).
// Inputs are copied once; the batch is integrated in ~64 MB output chunks on two
// streams so that the device->host copy of chunk i overlaps the integration of
// chunk i+1.  Device buffers and streams live in a per-device context that grows
// on demand and is reused by later calls (no cudaMalloc/cudaFree per call).
namespace {
struct HostCtx {
    std::mutex mu;
    bool init = false;
    cudaStream_t s[2] = {nullptr, nullptr};
    cudaEvent_t inputs_ready = nullptr;
    void *buf[11] = {nullptr};
    size_t cap[11] = {0};
    void *get(int k, size_t bytes, bool &ok)
    {
        if (bytes == 0) return nullptr;
        if (cap[k] < bytes) {
            if (buf[k]) cudaFree(buf[k]);
            buf[k] = nullptr;
            cap[k] = 0;
            if (cudaMalloc(&buf[k], bytes) != cudaSuccess) { ok = false; return nullptr; }
            cap[k] = bytes;
        }
        return buf[k];
    }
};
HostCtx g_host_ctx[64];
}  // namespace

int hxg_gram_batched_host(int space, int path, int p1, int p2, int p3, int L, int E,
                          const double *nodes, const double *weights, const int *kind,
                          const double *params, const double *coef, const double *wgrid,
                          double *out, int *status)
{
    int rc = check_common(space, path, p1, p2, p3, L, E);
    if (rc != HXG_OK) return rc;
    if (E == 0) return HXG_OK;
    if (!kind || !params || !out) return HXG_ERR_ARG;
    if ((nodes == nullptr) != (weights == nullptr)) return HXG_ERR_ARG;
    if (wgrid && path != GENERAL) return HXG_ERR_ARG;  // gram.py:93-98: constant weights only
    SpacePlan P;
    rc = build_plan(space, p1, p2, p3, P);
    if (rc != HXG_OK) return rc;
    const int Lt = path == AFFINE ? 1 : L;  // the affine kernels read only the F tables
    const bool user_rule = nodes && path != AFFINE;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return HXG_ERR_CUDA;
    HostCtx &cx = g_host_ctx[dev];
    std::lock_guard<std::mutex> lock(cx.mu);
    bool ok = true;
    auto chk = [&](cudaError_t e) { if (e != cudaSuccess) ok = false; };
    if (!cx.init) {
        chk(cudaStreamCreateWithFlags(&cx.s[0], cudaStreamNonBlocking));
        chk(cudaStreamCreateWithFlags(&cx.s[1], cudaStreamNonBlocking));
        chk(cudaEventCreateWithFlags(&cx.inputs_ready, cudaEventDisableTiming));
        if (!ok) return HXG_ERR_CUDA;
        cx.init = true;
    }
    const long long Pk = (long long)P.N * (P.N + 1) / 2;
    const size_t out_bytes_el = (size_t)Pk * sizeof(double);
    const size_t L3 = (size_t)L * L * L;
    long long chunk_bytes = 64ll << 20;  // D2H granularity: small chunks overlap the copy engine sooner
    if (const char *c = getenv("HXG_HOST_CHUNK_MB")) chunk_bytes = std::max(1ll, atoll(c)) << 20;  // tuning
    long long ch = std::max<long long>(1, chunk_bytes / (long long)out_bytes_el);
    ch = std::min<long long>(ch, E);
    size_t ws = hxg_workspace_size(space, path, p1, p2, p3, L, (int)ch);
    int *d_kind = (int *)cx.get(0, sizeof(int) * (size_t)E, ok);
    int *d_status = (int *)cx.get(1, sizeof(int) * (size_t)E, ok);
    double *d_params = (double *)cx.get(2, sizeof(double) * 24 * (size_t)E, ok);
    double *d_coef = coef ? (double *)cx.get(3, sizeof(double) * (size_t)E, ok) : nullptr;
    double *d_tab = (double *)cx.get(4, sizeof(double) * TAB_TOTAL, ok);
    double *d_out[2] = {(double *)cx.get(5, out_bytes_el * (size_t)ch, ok),
                        (double *)cx.get(6, out_bytes_el * (size_t)ch, ok)};
    void *d_ws[2] = {cx.get(7, ws, ok), cx.get(8, ws, ok)};
    double *d_wgrid = wgrid ? (double *)cx.get(9, sizeof(double) * L3 * (size_t)E, ok) : nullptr;
    double *d_rule = user_rule ? (double *)cx.get(10, sizeof(double) * 2 * (size_t)L, ok) : nullptr;
    if (!ok) return HXG_ERR_CUDA;
    cudaStream_t *s = cx.s;
    chk(cudaMemcpyAsync(d_kind, kind, sizeof(int) * (size_t)E, cudaMemcpyHostToDevice, s[0]));
    chk(cudaMemcpyAsync(d_params, params, sizeof(double) * 24 * (size_t)E, cudaMemcpyHostToDevice, s[0]));
    if (coef) chk(cudaMemcpyAsync(d_coef, coef, sizeof(double) * (size_t)E, cudaMemcpyHostToDevice, s[0]));
    if (wgrid) chk(cudaMemcpyAsync(d_wgrid, wgrid, sizeof(double) * L3 * (size_t)E, cudaMemcpyHostToDevice, s[0]));
    if (user_rule) {
        chk(cudaMemcpyAsync(d_rule, nodes, sizeof(double) * (size_t)L, cudaMemcpyHostToDevice, s[0]));
        chk(cudaMemcpyAsync(d_rule + L, weights, sizeof(double) * (size_t)L, cudaMemcpyHostToDevice, s[0]));
    }
    rc = hxg_make_tables(Lt, user_rule ? d_rule : nullptr, user_rule ? d_rule + L : nullptr, d_tab, s[0]);
    chk(cudaEventRecord(cx.inputs_ready, s[0]));
    chk(cudaStreamWaitEvent(s[1], cx.inputs_ready, 0));
    int i = 0;
    for (long long e0 = 0; e0 < E && ok && rc == HXG_OK; e0 += ch, ++i) {
        const int ne = (int)std::min<long long>(ch, E - e0);
        cudaStream_t st = s[i & 1];
        rc = hxg_gram_batched(space, path, p1, p2, p3, L, ne, d_kind + e0, d_params + 24 * e0,
                              d_coef ? d_coef + e0 : nullptr, d_wgrid ? d_wgrid + (size_t)e0 * L3 : nullptr,
                              d_tab, d_out[i & 1], d_status + e0, d_ws[i & 1], ws, st);
        if (rc != HXG_OK) break;
        chk(cudaMemcpyAsync(out + e0 * Pk, d_out[i & 1], out_bytes_el * (size_t)ne,
                            cudaMemcpyDeviceToHost, st));
    }
    chk(cudaStreamSynchronize(s[0]));
    chk(cudaStreamSynchronize(s[1]));
    if (rc != HXG_OK) return rc;
    if (!ok) return HXG_ERR_CUDA;
    // the reference raises before returning any matrix (geometry.py:214-223,
    // gram.py:170-174): flagged elements turn into an error code, with or without
    // a status array to say which
    std::vector<int> hs;
    int *st_host = status;
    if (!st_host) {
        hs.resize((size_t)E);
        st_host = hs.data();
    }
    if (cudaMemcpy(st_host, d_status, sizeof(int) * (size_t)E, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HXG_ERR_CUDA;
    int any = 0;
    for (int e = 0; e < E; ++e) any |= st_host[e];
    if (any & 2) return HXG_ERR_KIND;
    if (any & 1) return HXG_ERR_DEGENERATE;
    return HXG_OK;
}

}  // extern "C"
