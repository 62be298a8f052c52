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
