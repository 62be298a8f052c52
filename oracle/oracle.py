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
