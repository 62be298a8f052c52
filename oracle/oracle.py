"""ctypes front-end of the CPU oracle (oracle/hexgram_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs as the parity checker / CPU baseline.  The product
package never imports this module.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

SPACE_CODES = {"H1": 0, "Hcurl": 1, "Hdiv": 2, "L2": 3}
PATH_CODES = {"general": 0, "affine": 1, "extrusion": 2}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + pthreads)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_gauss_rule.argtypes = [ctypes.c_int, _dp, _dp]
        L.orc_shape1_h1.argtypes = [ctypes.c_double, ctypes.c_int, _dp, _dp]
        L.orc_shape1_l2.argtypes = [ctypes.c_double, ctypes.c_int, _dp]
        L.orc_ftable.argtypes = [ctypes.c_int, _dp]
        L.orc_dim.argtypes = [ctypes.c_int] * 4
        L.orc_geom_full.argtypes = [ctypes.c_int, _dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, _dp, _dp]
        L.orc_geom_full.restype = ctypes.c_double
        L.orc_gram_full.argtypes = [ctypes.c_int] * 6 + [_dp, _dp, ctypes.c_int, _dp,
                                                         ctypes.c_double, _dp, _dp]
        L.orc_gram_full.restype = ctypes.c_longlong
        L.orc_gram_batched.argtypes = [ctypes.c_int] * 7 + [_ip, _dp, _dp, _dp, _dp, ctypes.c_int]
        L.orc_num_cpus.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def num_cpus() -> int:
    return int(lib().orc_num_cpus())


def gauss_rule(L: int):
    n = np.zeros(32)
    w = np.zeros(32)
    if lib().orc_gauss_rule(L, _p(n), _p(w)) != 0:
        raise ValueError(f"bad rule order {L}")
    return n[:L].copy(), w[:L].copy()


def shape1_h1(xi: float, p: int):
    c = np.zeros(p + 1)
    d = np.zeros(p + 1)
    lib().orc_shape1_h1(xi, p, _p(c), _p(d))
    return c, d


def shape1_l2(xi: float, p: int):
    nu = np.zeros(max(p, 2))
    lib().orc_shape1_l2(xi, p, _p(nu))
    return nu[:p].copy()


def ftable(pmax: int):
    n = pmax + 1
    f = np.zeros((4, n, n))
    lib().orc_ftable(pmax, _p(f))
    return f


def geom_full(kind: int, params, xi):
    J = np.zeros((3, 3))
    Ji = np.zeros((3, 3))
    par = np.ascontiguousarray(params, dtype=np.float64)
    det = lib().orc_geom_full(kind, _p(par), xi[0], xi[1], xi[2], _p(J), _p(Ji))
    return J, Ji, det


def dim(space: str, orders) -> int:
    return int(lib().orc_dim(SPACE_CODES[space], *orders))


def gram_full(space: str, path: str, orders, L: int, kind: int, params, coef=1.0,
              wgrid=None, nodes=None, weights=None):
    """One element, full N x N matrix and the accumulation counter."""
    N = dim(space, orders)
    if nodes is None and path != "affine":
        nodes, weights = gauss_rule(L)
    nodes = np.ascontiguousarray(nodes if nodes is not None else np.zeros(1), dtype=np.float64)
    weights = np.ascontiguousarray(weights if weights is not None else np.zeros(1),
                                   dtype=np.float64)
    par = np.ascontiguousarray(params, dtype=np.float64)
    wg = None if wgrid is None else np.ascontiguousarray(wgrid, dtype=np.float64).reshape(-1)
    G = np.zeros((N, N))
    acc = lib().orc_gram_full(SPACE_CODES[space], PATH_CODES[path], orders[0], orders[1],
                              orders[2], L, _p(nodes), _p(weights), int(kind), _p(par),
                              float(coef), _p(wg), _p(G))
    if acc < 0:
        raise ValueError("oracle rejected the arguments")
    return G, int(acc)


def gram_batched(space: str, path: str, orders, L: int, kind, params, coef=None, wgrid=None,
                 nthreads: int = 0):
    """E elements -> packed upper triangles (E, N(N+1)/2), threads over elements."""
    kind = np.ascontiguousarray(kind, dtype=np.int32)
    E = kind.shape[0]
    params = np.ascontiguousarray(params, dtype=np.float64).reshape(E, 24)
    coef = None if coef is None else np.ascontiguousarray(coef, dtype=np.float64)
    wg = None if wgrid is None else np.ascontiguousarray(wgrid, dtype=np.float64)
    N = dim(space, orders)
    out = np.empty((E, N * (N + 1) // 2))
    rc = lib().orc_gram_batched(SPACE_CODES[space], PATH_CODES[path], orders[0], orders[1],
                                orders[2], L, E, kind.ctypes.data_as(_ip), _p(params),
                                _p(coef), _p(wg), _p(out), int(nthreads))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return out


def unpack(packed: np.ndarray, N: int) -> np.ndarray:
    """Packed row-major upper triangle -> full symmetric N x N."""
    iu = np.triu_indices(N)
    G = np.zeros((N, N))
    G[iu] = packed
    G.T[iu] = packed
    return G


# ---------------------------------------------------------------------------
# DPG-layer consumers of the Gram kernels, numpy
# restatements of /root/reference/pkg/src/hexgram/dpg.py
# ---------------------------------------------------------------------------
def _sep3(A1, A2, A3):
    """dpg.py:146-152: separable triple product, digit-lexicographic (fastest
    digit first) on both axes; products in einsum operand order."""
    T = (A1[:, None, None, :, None, None] * A2[None, :, None, None, :, None]) \
        * A3[None, None, :, None, None, :]
    # T[i, j, k, x, y, z] -> rows (k, j, i), columns (z, y, x)
    T = T.transpose(2, 1, 0, 5, 4, 3)
    r = A1.shape[0] * A2.shape[0] * A3.shape[0]
    c = A1.shape[1] * A2.shape[1] * A3.shape[1]
    return T.reshape(r, c)


def graph_mixed(pr: int, omega: float) -> np.ndarray:
    """dpg.py:155-176 _graph_mixed_ftables: S[ih, iv] = omega (q, div v) -
    omega (grad q, v) on the master element from the closed-form F01 table."""
    f01 = ftable(pr + 1)[1]
    q = pr + 1
    blocks = []
    for a in range(3):
        K1, K2 = [], []
        for d in range(3):
            n_d = q if d == a else pr
            sh = 0 if d == a else 1
            M1 = np.empty((q, n_d))
            M2 = np.empty((q, n_d))
            for i in range(q):
                for j in range(n_d):
                    M1[i, j] = f01[i, j + sh]
                    M2[i, j] = f01[j, i] if d == a else f01[i, j + sh]
            K1.append(M1)
            K2.append(M2)
        blocks.append(omega * (_sep3(*K1) - _sep3(*K2)))
    return np.hstack(blocks)


def adjoint_graph_gram(pr: int, omega: float, alpha: float, path: str, kind: int, params,
                       include_mixed: bool = True) -> np.ndarray:
    """dpg.py:179-231: real block form [[re, -im], [im, re]] with
    re = diag(G_H1, G_Hdiv) (mass weight omega^2 + alpha) and
    im = [[0, S], [-S^T, 0]]."""
    w = omega * omega + alpha
    L = pr + 1 if path != "affine" else 1
    o = (pr, pr, pr)
    Gq, _ = gram_full("H1", path, o, L, kind, params, coef=w)
    Gv, _ = gram_full("Hdiv", path, o, L, kind, params, coef=w)
    mw, mv = Gq.shape[0], Gv.shape[0]
    m = mw + mv
    re = np.zeros((m, m))
    re[:mw, :mw] = Gq
    re[mw:, mw:] = Gv
    im = np.zeros((m, m))
    if include_mixed:
        S = graph_mixed(pr, omega)
        im[:mw, mw:] = S
        im[mw:, :mw] = -S.T
    return np.block([[re, -im], [im, re]])


def condense(G: np.ndarray, B: np.ndarray, l: np.ndarray):
    """dpg.py:348-357: (B^T G^-1 B, B^T G^-1 l) through the lower Cholesky
    factor of G (cho_factor / cho_solve restated with numpy); raises
    numpy.linalg.LinAlgError when G is not positive definite."""
    from scipy.linalg import solve_triangular

    Lc = np.linalg.cholesky(G)
    X = solve_triangular(Lc.T, solve_triangular(Lc, B, lower=True), lower=False)
    y = solve_triangular(Lc.T, solve_triangular(Lc, l, lower=True), lower=False)
    return B.T @ X, B.T @ y


def mixed_tens_term(p0, pr, su, sh, geom_code, gr, gc, nodes, wts, kind, par):
    """_kernels.py:1861-1932 mixed_tens_term (numpy restatement, same stage
    order xi3 -> xi2 -> xi1): out[i_flat, k_flat] = integral of
    prod_d chi^(su_d)_{i_d+sh_d}(xi_d) nu_{k_d}(xi_d) g(xi), g by geom_code
    (0: 1, 1: 1/detJ, 2: J[gr,gc]/detJ, 3: Jinv[gr,gc])."""
    L = nodes.shape[0]
    n = [pr + 1 - s for s in sh]
    tab = []
    for l in range(L):
        c, d = shape1_h1(nodes[l], pr)
        nu = shape1_l2(nodes[l], p0)
        tab.append((c, d, nu))
    g = np.empty((L, L, L))
    for l in range(L):
        for m in range(L):
            for k in range(L):
                J, Ji, det = geom_full(kind, par, (nodes[l], nodes[m], nodes[k]))
                g[l, m, k] = (1.0, 1.0 / det, J[gr, gc] / det, Ji[gr, gc])[geom_code]
    U = []  # U[d][i, k, node] = chi^(su)_{i+sh}(x) nu_k(x) w(x)
    for dd in range(3):
        Ud = np.empty((n[dd], p0, L))
        for l in range(L):
            c, d, nu = tab[l]
            f = d if su[dd] == 1 else c
            Ud[:, :, l] = np.outer(f[sh[dd]:sh[dd] + n[dd]], nu) * wts[l]
        U.append(Ud)
    gA = np.einsum("lmn,ckn->lmck", g, U[2])           # xi3
    gB = np.einsum("lmck,bjm->lbjck", gA, U[1])        # xi2
    out = np.einsum("lbjck,ail->abcijk", gB, U[0])     # xi1: [i1, i2, i3, k1, k2, k3]
    nt = n[0] * n[1] * n[2]
    # flat indices: i1 + n1 (i2 + n2 i3), k1 + p0 (k2 + p0 k3)
    return out.transpose(2, 1, 0, 5, 4, 3).reshape(nt, p0 ** 3)


def acoustics_stiffness(p0, pr, omega, kind, par):
    """dpg.py:234-277 _acoustics_b_tensorized: (Bre, Bim) with the L = pr + 1 rule."""
    nodes, wts = gauss_rule(pr + 1)
    mw = (pr + 1) ** 3
    mv = dim("Hdiv", (pr, pr, pr))
    ny = p0 ** 3
    Bre = np.zeros((mw + mv, 4 * ny))
    Bim = np.zeros((mw + mv, 4 * ny))
    T = lambda su, sh, gc, r, c: mixed_tens_term(p0, pr, su, sh, gc, r, c, nodes, wts, kind, par)  # noqa: E731
    Bim[:mw, :ny] += omega * T((0, 0, 0), (0, 0, 0), 0, 0, 0)
    for d in range(3):
        su = tuple(1 if e == d else 0 for e in range(3))
        for c in range(3):
            Bre[:mw, ny * (1 + c):ny * (2 + c)] -= T(su, (0, 0, 0), 3, d, c)
    off = mw
    for a in range(3):
        sh = tuple(0 if e == a else 1 for e in range(3))
        na = (pr + 1 - sh[0]) * (pr + 1 - sh[1]) * (pr + 1 - sh[2])
        Bre[off:off + na, :ny] -= T((1, 1, 1), sh, 1, 0, 0)
        su = tuple(0 if e == a else 1 for e in range(3))
        for c in range(3):
            Bim[off:off + na, ny * (1 + c):ny * (2 + c)] += omega * T(su, sh, 2, c, a)
        off += na
    return Bre, Bim


def acoustics_load(p0, pr, kind, par, fgrid, pairing="velocity"):
    """dpg.py:280-302 _acoustics_load (real part over the stacked test space);
    fgrid = the source at the tensor nodes (l, m, n) of the L = pr + 1 rule."""
    L = pr + 1
    nodes, wts = gauss_rule(L)
    q = pr + 1
    mw = q ** 3
    nb = q * pr * pr
    lre = np.zeros(mw + 3 * nb)
    if fgrid is None:
        return lre
    fg = np.asarray(fgrid).reshape(L, L, L)
    C = [shape1_h1(x, pr)[0] for x in nodes]
    NU = [shape1_l2(x, pr)[:pr] for x in nodes]
    for l in range(L):
        for m in range(L):
            for k in range(L):
                J, _, det = geom_full(kind, par, (nodes[l], nodes[m], nodes[k]))
                w = wts[l] * wts[m] * wts[k] * fg[l, m, k]
                pts = (l, m, k)
                if pairing == "pressure":
                    phi = np.einsum("i,j,k->kji", C[l], C[m], C[k]).reshape(-1)
                    lre[:mw] += phi * (w * det)
                else:
                    Jrows = J.sum(axis=0)
                    off = mw
                    for a in range(3):
                        f = [C[pts[d]] if d == a else NU[pts[d]] for d in range(3)]
                        v = np.einsum("i,j,k->kji", f[0], f[1], f[2]).reshape(-1)
                        lre[off:off + nb] += w * Jrows[a] * v
                        off += nb
    return lre
