"""Device versions of the two direct consumers of the Gram kernels in the
reference's DPG layer (/root/reference/pkg/src/hexgram/dpg.py; SURVEY 8(f)
rows 2 and 3):

* ``adjoint_graph_gram`` (dpg.py:179-231) -- the ultraweak-acoustics test
  Gram over H1 x H(div): the H1 and H(div) Grams with mass weight
  omega^2 + alpha (the batched Gram kernels, ``coef``), the closed-form
  frequency coupling S (dpg.py:155-176, ``hxg_graph_mixed``) and the real
  block form [[re, -im], [im, re]] (dpg.py:205-219, ``hxg_graph_assemble``);
* ``condense`` (dpg.py:348-357) -- static condensation A = B^T G^-1 B,
  rhs = B^T G^-1 l through a Cholesky factorisation of G
  (``hxg_condense_batched``);
* ``acoustics_ultraweak_element`` (dpg.py:305-336) -- the ultraweak
  acoustics element system: G from the adjoint-graph Gram, the
  sum-factorized stiffness B (dpg.py:234-277, mixed_tens_term) and the load
  l (dpg.py:280-302) in real block form (``hxg_acoustics_batched``).

The per-element functions keep the reference's names, arguments, errors and
return types; the ``*_batched`` functions are the native entries (device
tensors, packed Gram layout).  Every floating-point operation runs in the
sm_100a kernels of libhexgram_b200.so; there is no CPU fallback.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from .errors import NonSPDError, SimplificationNotApplicableError
from .geometry import ElementMap, classify, map_position
from .gram import GramResult, OpCounters, counters
from .spaces import SpaceSignature, dim

__all__ = [
    "DpgElementSystem",
    "UltraweakAcousticsProblem",
    "acoustics_ultraweak_element",
    "acoustics_batched",
    "graph_mixed_block",
    "adjoint_graph_gram",
    "adjoint_graph_gram_batched",
    "condense",
    "condense_batched",
]


def _engine(device=None):
    from .engine import get_engine

    return get_engine(device)


def _vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(eng, stream=None):
    st = stream or torch.cuda.current_stream(eng.device)
    return st, ctypes.c_void_p(st.cuda_stream)


def graph_mixed_block(p_r: int, omega: float, *, device=None, stream=None) -> torch.Tensor:
    """Adjoint-graph cross block S [(p_r+1)^3, 3 p_r^2 (p_r+1)] on the device
    (dpg.py:155-176 ``_graph_mixed_ftables``)."""
    from .engine import _check

    eng = _engine(device)
    st, sp = _stream(eng, stream)
    q = p_r + 1
    S = torch.empty((q ** 3, 3 * p_r * p_r * q), dtype=torch.float64, device=eng.device)
    tab = eng.tables(q, stream=st)
    _check(eng.lib.hxg_graph_mixed(int(p_r), float(omega), _vp(tab), _vp(S), sp), "hxg_graph_mixed")
    return S


def _graph_paths(backend: str, emap_class: str | None):
    if backend in ("conventional", "tensorized"):
        return "general"
    if backend == "simplified":
        if emap_class == "general":
            raise SimplificationNotApplicableError(
                "map class 'general' admits no simplification")
        return "affine" if emap_class == "constant-jacobian" else "extrusion"
    raise ValueError(f"unknown backend {backend!r}")


def adjoint_graph_gram_batched(p_r: int, omega: float, alpha: float, kind, params, *,
                               path: str = "general", include_mixed: bool = True,
                               layout: str = "packed", device=None, stream=None):
    """Batched adjoint-graph Gram in real block form (dpg.py:179-231) for E
    elements: kind int32 [E], params float64 [E, 24] (device tensors or host
    arrays); ``path`` as in ``gram_batched``.  Returns a device tensor
    [E, 2m(2m+1)/2] (``layout="packed"``, row-major upper triangles, the
    input layout of ``condense_batched``) or [E, 2m, 2m] (``"full"``),
    m = (p_r+1)^3 + 3 p_r^2 (p_r+1)."""
    from .engine import _check

    if omega <= 0 or alpha <= 0:
        raise ValueError("omega and alpha must be positive")
    if layout not in ("packed", "full"):
        raise ValueError("layout must be 'packed' or 'full'")
    eng = _engine(device)
    st, sp = _stream(eng, stream)
    w = omega * omega + alpha
    L = p_r + 1
    orders = (p_r, p_r, p_r)
    kind = torch.as_tensor(kind, dtype=torch.int32).to(eng.device)
    E = int(kind.shape[0])
    coef = torch.full((E,), w, dtype=torch.float64, device=eng.device)
    Lp = 1 if path == "affine" else L
    gq, _ = eng.integrate("H1", path, orders, Lp, kind, params, coef, stream=st)
    gv, _ = eng.integrate("Hdiv", path, orders, Lp, kind, params, coef, stream=st)
    S = graph_mixed_block(p_r, omega, device=eng.device, stream=st) if include_mixed else None
    m = dim(SpaceSignature("H1", orders)) + dim(SpaceSignature("Hdiv", orders))
    M2 = 2 * m
    if layout == "full":
        out = torch.empty((E, M2, M2), dtype=torch.float64, device=eng.device)
        rc = eng.lib.hxg_graph_assemble(p_r, E, _vp(gq), _vp(gv), _vp(S), _vp(out), None, sp)
    else:
        out = torch.empty((E, M2 * (M2 + 1) // 2), dtype=torch.float64, device=eng.device)
        rc = eng.lib.hxg_graph_assemble(p_r, E, _vp(gq), _vp(gv), _vp(S), None, _vp(out), sp)
    _check(rc, "hxg_graph_assemble")
    return out


def adjoint_graph_gram(p_r: int, omega: float, alpha: float, emap: ElementMap,
                       backend: str = "conventional", include_mixed: bool = True) -> GramResult:
    """Adjoint-graph Gram over W^{p_r} x V^{p_r} in real block form
    (dpg.py:179-231), one element, on the device.  The cross block is the
    closed-form S for every backend (the reference's conventional backend
    integrates the same master-element polynomial exactly by quadrature,
    dpg.py:191-199)."""
    if omega <= 0 or alpha <= 0:
        raise ValueError("omega and alpha must be positive")
    klass = classify(emap)
    path = _graph_paths(backend, klass)
    full = adjoint_graph_gram_batched(p_r, omega, alpha, np.array([emap.kind_code], np.int32),
                                      emap.params.reshape(1, 24), path=path,
                                      include_mixed=include_mixed, layout="full")
    G = full[0].cpu().numpy()
    orders = (p_r, p_r, p_r)
    L = p_r + 1
    if backend == "simplified":
        ex = klass == "extrusion"
        cq = counters("H1", orders, "simplified", L if ex else None,
                      klass="extrusion" if ex else "constant-jacobian")
        cv = counters("Hdiv", orders, "simplified", L if ex else None,
                      klass="extrusion" if ex else "constant-jacobian")
    else:
        cq = counters("H1", orders, backend, L)
        cv = counters("Hdiv", orders, backend, L)
    cnt = OpCounters(cq.accumulations + cv.accumulations, cq.geometry_calls + cv.geometry_calls,
                     cq.shape1_calls + cv.shape1_calls, cq.shape3_calls + cv.shape3_calls)
    return GramResult(G, cnt)


def condense_batched(G, B, l=None, *, device=None, stream=None, check: bool = True):
    """Batched static condensation (dpg.py:348-357): per element
    A = B^T G^-1 B [n, n] and rhs = B^T G^-1 l [n].  G: packed upper triangles
    [E, m(m+1)/2] (the Gram kernels' layout); B [E, m, n]; l [E, m] or None.
    Device tensors or host arrays.  Returns (A, rhs, status) device tensors;
    raises NonSPDError if a G is not positive definite (``check``)."""
    from .engine import _check

    eng = _engine(device)
    st, sp = _stream(eng, stream)
    dev = eng.device
    B = torch.as_tensor(B, dtype=torch.float64).to(dev).contiguous()
    if B.dim() != 3:
        raise ValueError("B must be [E, m, n]")
    E, m, n = (int(x) for x in B.shape)
    G = torch.as_tensor(G, dtype=torch.float64).to(dev)
    if G.numel() != E * (m * (m + 1) // 2):
        raise ValueError("G must hold m(m+1)/2 packed entries per element")
    G = G.reshape(E, m * (m + 1) // 2).contiguous()
    if l is not None:
        l = torch.as_tensor(l, dtype=torch.float64).to(dev).reshape(E, m).contiguous()
    A = torch.empty((E, n, n), dtype=torch.float64, device=dev)
    rhs = torch.empty((E, n), dtype=torch.float64, device=dev)
    status = torch.zeros(E, dtype=torch.int32, device=dev)
    ws_bytes = eng.lib.hxg_condense_workspace_size(m, n, max(E, 1))
    with eng._lock:
        ws = eng.workspace(ws_bytes, st)
        rc = eng.lib.hxg_condense_batched(m, n, E, _vp(G), _vp(B), _vp(l), _vp(A), _vp(rhs),
                                          _vp(status), _vp(ws), ws_bytes, sp)
    _check(rc, "hxg_condense_batched")
    if check:
        bad = torch.nonzero(status).flatten()
        if bad.numel():
            raise NonSPDError(f"Gram matrix not SPD during condensation (element {int(bad[0])})")
    return A, rhs, status


def condense(system):
    """Static condensation to (B^T G^-1 B, B^T G^-1 l) (dpg.py:348-357) for one
    element system (any object with ``G``, ``B``, ``l``; the reference's
    DpgElementSystem), on the device; sets ``system.condensed``."""
    G = np.asarray(system.G, dtype=np.float64)
    m = G.shape[0]
    packed = G[np.triu_indices(m)]
    B = np.asarray(system.B, dtype=np.float64)
    l = np.asarray(system.l, dtype=np.float64)
    A, rhs, _ = condense_batched(packed[None], B[None], l[None])
    A = A[0].cpu().numpy()
    rhs = rhs[0].cpu().numpy()
    system.condensed = (A, rhs)
    return A, rhs


# ---------------------------------------------------------------------------
# ultraweak acoustics element system (dpg.py:44-92, 234-336)
# ---------------------------------------------------------------------------
@dataclass
class DpgElementSystem:
    """Arrays of the enriched element system G s - B u = -l (dpg.py:44-75)."""

    G: np.ndarray
    B: np.ndarray
    l: np.ndarray
    orders: tuple
    is_complex: bool = False
    condensed: tuple | None = None
    gram_counters: OpCounters | None = None

    def __post_init__(self):
        m = self.B.shape[0]
        n = self.B.shape[1]
        if self.is_complex:
            m //= 2
            n //= 2
        if m <= n:
            raise ValueError(f"enriched test space must dominate: m={m} <= n={n}")

    @property
    def m(self) -> int:
        return self.B.shape[0] // (2 if self.is_complex else 1)

    @property
    def n(self) -> int:
        return self.B.shape[1] // (2 if self.is_complex else 1)


@dataclass(frozen=True)
class UltraweakAcousticsProblem:
    """Frequency, broken-norm correction and source (dpg.py:78-92)."""

    omega: float
    alpha: float
    f: object = None
    load_pairing: str = "velocity"

    def __post_init__(self):
        if self.omega <= 0:
            raise ValueError("omega must be positive")
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if self.load_pairing not in ("velocity", "pressure"):
            raise ValueError("load_pairing must be 'velocity' or 'pressure'")


def acoustics_batched(p0: int, pr: int, omega: float, kind, params, fgrid=None, *,
                      pairing: str = "velocity", block_form: bool = True, parts: bool = True,
                      device=None, stream=None):
    """Batched ultraweak-acoustics stiffness (dpg.py:234-277) and load
    (dpg.py:280-302) on the device, rule L = pr + 1.  kind int32 [E], params
    float64 [E, 24]; fgrid float64 [E, L^3] (source at the tensor nodes, point
    (l, m, n) -> (l L + m) L + n) or None.  Returns (Bre [E, m, n],
    Bim [E, m, n] (None unless ``parts``), B2 [E, 2m, 2n] (None unless
    ``block_form``), l [E, 2m] or None, status)."""
    if not (parts or block_form):
        raise ValueError("request at least one of parts / block_form")
    from .engine import _check

    eng = _engine(device)
    st, sp = _stream(eng, stream)
    dev = eng.device
    L = pr + 1
    kind = torch.as_tensor(kind, dtype=torch.int32).to(dev).contiguous()
    E = int(kind.shape[0])
    params = torch.as_tensor(params, dtype=torch.float64).to(dev).reshape(E, 24).contiguous()
    q = pr + 1
    m = q ** 3 + 3 * pr * pr * q
    n = 4 * p0 ** 3
    Bre = torch.empty((E, m, n), dtype=torch.float64, device=dev) if parts else None
    Bim = torch.empty((E, m, n), dtype=torch.float64, device=dev) if parts else None
    B2 = torch.empty((E, 2 * m, 2 * n), dtype=torch.float64, device=dev) if block_form else None
    lre = None
    if fgrid is not None:
        fgrid = torch.as_tensor(fgrid, dtype=torch.float64).to(dev).reshape(E, L ** 3).contiguous()
        lre = torch.empty((E, 2 * m), dtype=torch.float64, device=dev)
    status = torch.zeros(E, dtype=torch.int32, device=dev)
    tab = eng.tables(L, stream=st)
    ws_bytes = eng.lib.hxg_acoustics_workspace_size(p0, pr, L, E)
    with eng._lock:
        ws = eng.workspace(ws_bytes, st)
        rc = eng.lib.hxg_acoustics_batched(p0, pr, float(omega), L, E, _vp(kind), _vp(params),
                                           _vp(tab), _vp(fgrid), 0 if pairing == "velocity" else 1,
                                           _vp(Bre), _vp(Bim), _vp(B2), _vp(lre), _vp(status),
                                           _vp(ws), ws_bytes, sp)
    _check(rc, "hxg_acoustics_batched")
    return Bre, Bim, B2, lre, status


def _source_grid(fun, emap: ElementMap, L: int) -> np.ndarray | None:
    """The source sampled at the tensor nodes, as dpg.py:95-103 does on the host."""
    if fun is None:
        return None
    from .quadrature import tensor_rule

    pts = tensor_rule(L).points
    if np.isscalar(fun):
        return np.full(pts.shape[0], float(fun))
    return np.array([float(fun(map_position(emap, p))) for p in pts])


def acoustics_ultraweak_element(problem: UltraweakAcousticsProblem, p0: int, dp: int,
                                emap: ElementMap, backend: str = "tensorized") -> DpgElementSystem:
    """Ultraweak acoustics element arrays in real block form (dpg.py:305-336),
    on the device: G = adjoint_graph_gram(pr, omega, alpha, emap, backend), B
    by sum factorization (both the reference's routes give the same integral),
    l from the source sampled at the tensor nodes."""
    if p0 < 1 or dp < 1:
        raise ValueError("p0 and dp must be >= 1")
    pr = p0 + dp
    L = pr + 1
    gres = adjoint_graph_gram(pr, problem.omega, problem.alpha, emap, backend)
    fg = _source_grid(problem.f, emap, L)
    _, _, B2, lre, status = acoustics_batched(
        p0, pr, problem.omega, np.array([emap.kind_code], np.int32), emap.params.reshape(1, 24),
        None if fg is None else fg[None], pairing=problem.load_pairing, parts=False)
    B = B2[0].cpu().numpy()
    m = B.shape[0] // 2
    l = lre[0].cpu().numpy() if lre is not None else np.zeros(2 * m)
    return DpgElementSystem(G=gres.matrix, B=B, l=l, orders=(p0, dp, pr), is_complex=True,
                            gram_counters=gres.counters)
