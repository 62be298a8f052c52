/*
 * hexgram_b200.h -- C ABI of the B200 (sm_100a) Gram-integration library
 * libhexgram_b200.so.
 *
 * This is the drop-in seam for the reference's compiled kernels.  In the
 * reference (/root/reference/pkg/src/hexgram) control enters compiled code
 * at the numba dispatchers selected in gram.py:
 *
 *   gram.py:127-136  _TENS_KERNELS[(space, loop_order)] ->
 *                    tens_{l2,h1,hdiv,hcurl}_{std,alt}(p1,p2,p3,nodes,wts,kind,par,wgrid)
 *                    (_kernels.py:356-1150), called at gram.py:154-157
 *   gram.py:183-191  simp_{l2,h1,hdiv,hcurl}_const(p1,p2,p3,fall,kind,par,wmass)
 *                    (_kernels.py:1169-1404)
 *
 * Each reference call integrates ONE element and returns a dense N x N
 * matrix plus operation counters.  The entry points below integrate a BATCH
 * of E independent elements per call (the reference's calls are pure and
 * independent), writing packed upper triangles.
 *
 * Conventions
 *   space  : 0 = H1, 1 = H(curl), 2 = H(div), 3 = L2   (spaces.py:30 order differs;
 *            the codes here are the library's own)
 *   path   : 0 = general map, sum factorization O(p^7)  (gram_tensorized)
 *            1 = constant-Jacobian map, O(p^6)           (gram_simplified, kinds 0..2)
 *            2 = extrusion map, O(p^6): F tables in xi1, L x L rule in (xi2, xi3)
 *                at xi1 = 0.5                            (gram_simplified, kinds 0..3)
 *   kind   : element-map kind codes of geometry.py:46-52
 *            (0 identity, 1 diagonal-affine, 2 general-affine, 3 extrusion, 4 trilinear)
 *   params : 24 doubles per element, layout of geometry.py:83-119
 *   coef   : per-element scalar weight of the mass (zeroth-order) term only
 *            (gram.py:66-98, _kernels.py:15-18); may be NULL (= 1)
 *   wgrid  : optional per-element, per-quadrature-node mass weight
 *            [E][L][L][L] (gram.py:78-90 sampled on the host); general path only;
 *            overrides coef when non-NULL
 *   out    : [E][N(N+1)/2] fp64, row-major packed upper triangle
 *            (entry (r,c), r <= c, at r*N - r*(r-1)/2 + (c-r))
 *   status : [E] int bit mask, written by the call: 0 ok; bit 0: det J <= 0 at
 *            an evaluated point (the reference raises DegenerateMapError,
 *            errors.py:12-20); bit 1: simplified path asked for a map kind it
 *            does not cover -- > 2 on path 1, > 3 on path 2
 *            (SimplificationNotApplicableError, gram.py:170-174)
 *
 * All pointers of hxg_gram_batched are DEVICE pointers; the call is
 * stream-ordered, does no host synchronisation and is safe to issue from
 * several host threads on distinct streams.  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Return values are HXG_OK or a negative
 * HXG_ERR_* code; the Python layer maps them onto the reference's exception
 * types (errors.py).
 */
#ifndef HEXGRAM_B200_H
#define HEXGRAM_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    HXG_OK = 0,
    HXG_ERR_ORDER = -1,        /* InvalidOrderError: p_d < 1, p_d > HXG_MAX_ORDER, bad L */
    HXG_ERR_SPACE = -2,        /* unknown space / path code                                */
    HXG_ERR_KIND = -3,         /* SimplificationNotApplicableError (gram.py:171-174)       */
    HXG_ERR_WORKSPACE = -4,    /* workspace too small                                      */
    HXG_ERR_CUDA = -5,         /* CUDA launch / runtime error                              */
    HXG_ERR_ARG = -6,          /* NULL pointer or negative count                           */
    HXG_ERR_DEGENERATE = -7    /* host entry: an element has det J <= 0 (DegenerateMapError,
                                  errors.py:12-20)                                          */
};

#define HXG_MAX_ORDER 12   /* poly1d.py:37 DEFAULT_P_MAX, cli.py:55 MAX_SUPPORTED_ORDER */
#define HXG_MAX_RULE 16    /* 1D Gauss points supported by the device kernels           */

/* library version, e.g. 100 for 0.1.0 */
int hxg_version(void);

/* Highest isotropic order p (rule L = p + 1) for which hxg_gram_batched(path = 0) runs as
 * one kernel that evaluates the element geometry itself -- no hxg_metric_batched pass and
 * no workspace.  hxg_metric_batched + hxg_contract_batched remain valid at every order. */
int hxg_fused_order_max(void);
const char *hxg_error_string(int code);

/* spaces.py:67-80 -- number of basis functions N; <0 on bad arguments */
int hxg_dim(int space, int p1, int p2, int p3);

/* OpCounters.accumulations of the reference for the same call
 * (closed forms; gram.py:45-50) */
long long hxg_accumulations(int space, int path, int p1, int p2, int p3, int L);

/* Size in doubles of the device 1D-table block used by hxg_gram_batched. */
size_t hxg_tables_doubles(void);

/* Build the 1D tables on the device (quadrature.py:47-66, _kernels.py:29-53,
 * poly1d.py:140-266): Gauss-Legendre nodes/weights on (0,1) for L points,
 * chi_k / chi'_k at the nodes, and the closed-form F tables.  If `nodes` and
 * `weights` (device pointers, L each) are non-NULL they are used instead of
 * the Gauss rule (a user-supplied Rule1D, gram.py:139-151). */
int hxg_make_tables(int L, const double *nodes, const double *weights, double *tables,
                    void *stream);

/* Device workspace (bytes) needed by hxg_gram_batched for this call. */
size_t hxg_workspace_size(int space, int path, int p1, int p2, int p3, int L, int E);

/* Batched Gram integration -- replaces tens_*_{std,alt} (path 0),
 * simp_*_const (path 1, _kernels.py:1169-1404) and simp_*_ext (path 2,
 * _kernels.py:1405-1764).  tables from hxg_make_tables(L, ...) (path 1: any L). */
int hxg_gram_batched(int space, int path, int p1, int p2, int p3, int L, int E,
                     const int *kind, const double *params, const double *coef,
                     const double *wgrid, const double *tables, double *out, int *status,
                     void *workspace, size_t workspace_bytes, void *stream);

/* The two stages of the general path, exported separately so callers can
 * schedule / time them (hxg_gram_batched = metric + contract per chunk).
 * hxg_metric_batched: per-point metric kernel, metric[E][nfields][L^3]
 *   (Jacobian, det, D, C, weights and mass coefficient folded; _kernels.py:56-136
 *   and the per-point weight folding of tens_*, e.g. _kernels.py:578-590).
 *   metric must hold hxg_workspace_size(space, 0, p.., L, E) bytes for this E.
 * hxg_contract_batched: three-stage sum-factorized contraction + packed output
 *   writer (stages A/B/C of tens_*_alt, _kernels.py:541-624, 742-853, 1003-1150). */
int hxg_metric_batched(int space, int p1, int p2, int p3, int L, int E, const int *kind,
                       const double *params, const double *coef, const double *wgrid,
                       const double *tables, double *metric, int *status, void *stream);
int hxg_contract_batched(int space, int p1, int p2, int p3, int L, int E, const double *tables,
                         const double *metric, double *out, void *stream);

/* Same computation with HOST inputs and HOST output: the reference's calling
 * convention at the kernel seam gram.py:154-157,
 *     kern(p1, p2, p3, rule1d.nodes, rule1d.weights, kind, params, wgrid)
 * (numpy in, numpy out), batched over E elements.  Copies the inputs in,
 * integrates in device-sized chunks and streams the packed triangles back,
 * overlapping the device->host copies with the next chunk's integration.
 *   nodes, weights : host [L] 1D rule on (0,1) (a user Rule1D), or both NULL for
 *                    the L-point Gauss rule (quadrature.py:47-66); ignored on path 1
 *   coef           : host [E] constant mass weights, or NULL (= 1)
 *   wgrid          : host [E][L][L][L] mass weight sampled at the tensor nodes
 *                    (gram.py:78-90, a callable mass_weight), or NULL; general path
 *                    only (the simplified paths take constants, gram.py:93-98:
 *                    HXG_ERR_ARG otherwise); overrides coef
 *   out            : host [E][N(N+1)/2]; page-locked for full copy bandwidth
 *   status         : host [E] or NULL; per-element flags as hxg_gram_batched
 * Synchronous.  Like the reference, which raises before returning a matrix, a
 * flagged element makes the call return HXG_ERR_KIND (bit 1) or
 * HXG_ERR_DEGENERATE (bit 0) -- whether or not `status` is given. */
int hxg_gram_batched_host(int space, int path, int p1, int p2, int p3, int L, int E,
                          const double *nodes, const double *weights, const int *kind,
                          const double *params, const double *coef, const double *wgrid,
                          double *out, int *status);

/* Expand packed upper triangles [E][N(N+1)/2] into full symmetric
 * matrices [E][N][N] on the device (the reference's GramResult.matrix
 * layout, gram.py:53-56, mirrored as _kernels.py:161-174 does). */
int hxg_expand_full(int N, int E, const double *packed, double *full, void *stream);


/* ------------------------------------------------------------------------
 * Direct consumers of the Gram kernels in the reference's DPG layer
 * (/root/reference/pkg/src/hexgram/dpg.py).
 * All pointers are DEVICE pointers; stream-ordered, no host sync.
 * ------------------------------------------------------------------------ */

/* dpg.py:155-176 _graph_mixed_ftables: the adjoint-graph cross block
 * S[mw][mv] (row-major), mw = (pr+1)^3 (H1 test space), mv = 3 pr^2 (pr+1)
 * (H(div) test space), S[ih][iv] = omega ((q_i, div v_j) - (grad q_i, v_j))
 * on the master element, from the closed-form F tables of `tables`
 * (hxg_make_tables, any L). */
int hxg_graph_mixed(int pr, double omega, const double *tables, double *S, void *stream);

/* dpg.py:205-219 adjoint_graph_gram: real block form [[re, -im], [im, re]] of
 * the adjoint-graph Gram, re = diag(Gq, Gv), im = [[0, S], [-S^T, 0]], for E
 * elements from the packed H1 Gram g_h1 [E][mw(mw+1)/2] and H(div) Gram
 * g_hdiv [E][mv(mv+1)/2] (hxg_gram_batched with coef = omega^2 + alpha) and
 * S (NULL: include_mixed=False).  Writes full [E][2m][2m] (m = mw + mv)
 * and/or packed [E][2m(2m+1)/2] row-major upper triangles (either may be
 * NULL, not both). */
int hxg_graph_assemble(int pr, int E, const double *g_h1, const double *g_hdiv, const double *S,
                       double *full, double *packed, void *stream);

/* Workspace (bytes) hxg_condense_batched wants for E elements of sizes m, n
 * (it works in chunks; one element's (m+n+1)^2 doubles is the minimum). */
size_t hxg_condense_workspace_size(int m, int n, int E);

/* dpg.py:348-357 condense, batched: per element A = B^T G^-1 B [n][n] and
 * rhs = B^T G^-1 l [n] through a Cholesky factorisation of G (partial
 * Cholesky elimination of [[G, B, l], [B^T, 0], [l^T, 0]], FP64).
 *   G   : [E][m(m+1)/2] packed upper triangles (the hxg_gram_batched layout)
 *   B   : [E][m][n] row-major;  l : [E][m] or NULL (rhs = 0)
 *   A   : [E][n][n];  rhs : [E][n] or NULL
 *   status : [E] or NULL; bit 2 (value 4) set when a pivot of G is not
 *            positive (the reference raises NonSPDError, dpg.py:350-353). */
int hxg_condense_batched(int m, int n, int E, const double *G, const double *B, const double *l,
                         double *A, double *rhs, int *status, void *workspace, size_t workspace_bytes,
                         void *stream);

/* Workspace (bytes) of hxg_acoustics_batched: per-point geometry fields. */
size_t hxg_acoustics_workspace_size(int p0, int pr, int L, int E);

/* dpg.py:234-277 _acoustics_b_tensorized (+ _kernels.py:1861-1936
 * mixed_tens_term) and dpg.py:280-302 _acoustics_load, batched: the
 * ultraweak-acoustics stiffness of E elements, trial order p0 (pressure + 3
 * velocity components, each p0^3 L2 functions, n = 4 p0^3 columns), test
 * order pr (H1 then H(div) rows, m = (pr+1)^3 + 3 pr^2 (pr+1)), L-point rule
 * (tables from hxg_make_tables(L)).
 *   Bre, Bim : [E][m][n] real / imaginary parts (row-major), or both NULL
 *   B2       : [E][2m][2n] real block form [[Bre, -Bim], [Bim, Bre]] or NULL
 *              (at least one of the two forms)
 *   fgrid    : [E][L^3] source sampled at the tensor nodes (l, m, n), or NULL
 *   lre      : [E][2m] load in real block form [l_re; 0], or NULL
 *   pairing  : 0 velocity (the printed form), 1 pressure (dpg.py:83-90)
 *   status   : [E] or NULL, bit 0: det J <= 0 at a quadrature point */
int hxg_acoustics_batched(int p0, int pr, double omega, int L, int E, const int *kind,
                          const double *params, const double *tables, const double *fgrid, int pairing,
                          double *Bre, double *Bim, double *B2, double *lre, int *status,
                          void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEXGRAM_B200_H */
