"""Drop-in Gram entry points (the surface of
/root/reference/pkg/src/hexgram/gram.py), served by the sm_100a kernels.

Per-element calls (`gram_tensorized`, `gram_simplified`, `gram`,
`gram_block`) keep the reference's names, signatures, argument meaning,
defaults, error behaviour and return type (`GramResult` with a full N x N
float64 matrix and exact `OpCounters`).  `gram_batched` is the native
batched entry: device tensors in, packed upper triangles out.

Both loop orders of the reference give identical matrices
(test_gram.py:103-112); the device path has one algorithm, so `loop_order`
only selects which reference counters are reported.
"""

from dataclasses import dataclass

import numpy as np

from .errors import NonSPDError, SimplificationNotApplicableError
from .geometry import ElementMap, classify, map_position
from .poly1d import FTable
from .quadrature import Rule1D, Rule3D, default_rule_order, gauss_rule
from .spaces import SpaceSignature, dim

__all__ = [
    "OpCounters",
    "GramResult",
    "BACKENDS",
    "gram_conventional",
    "gram_tensorized",
    "gram_simplified",
    "gram_block",
    "gram",
    "gram_batched",
    "counters",
]

BACKENDS = ("conventional", "tensorized", "simplified")


@dataclass(frozen=True)
class OpCounters:
    accumulations: int
    geometry_calls: int
    shape1_calls: int
    shape3_calls: int


@dataclass(frozen=True)
class GramResult:
    matrix: np.ndarray
    counters: OpCounters

    def cholesky(self) -> np.ndarray:
        try:
            return np.linalg.cholesky(self.matrix)
        except np.linalg.LinAlgError as exc:
            raise NonSPDError(f"Gram matrix is not positive definite: {exc}")


# ---------------------------------------------------------------------------
# reference operation counters, closed forms (verified against the reference
# kernels by tests/test_counters.py)
# ---------------------------------------------------------------------------
def _pairs3(space: str, orders) -> int:
    p3 = orders[2]
    if space == "L2":
        return p3 * (p3 + 1) // 2
    if space == "H1":
        return (p3 + 1) * (p3 + 2) // 2
    return (p3 + 1) ** 2


def _acc(space: str, orders, L: int | None) -> int:
    N = dim(SpaceSignature(space, orders))
    if space == "L2":
        t = 1
        for p in orders:
            t *= p * (p + 1) // 2
        return t if L is None else L * t
    T = {"H1": 10, "Hcurl": 5, "Hdiv": 2}[space]
    tri = N * (N + 1) // 2
    return T * tri if L is None else T * L * tri


def counters(space: str, orders, backend: str, L: int | None = None,
             loop_order: str = "alternative", klass: str = "constant-jacobian") -> OpCounters:
    orders = tuple(orders)
    if backend == "conventional":
        N = dim(SpaceSignature(space, orders))
        return OpCounters(L ** 3 * N * (N + 1) // 2, L ** 3, 0, L ** 3)
    if backend == "tensorized":
        if loop_order == "alternative":
            return OpCounters(_acc(space, orders, L), L ** 3, L + L * L + L ** 3, 0)
        pr = _pairs3(space, orders)
        return OpCounters(_acc(space, orders, L), L ** 3 * pr, L * (1 + pr * (L + L * L)), 0)
    if klass == "extrusion":
        pr = _pairs3(space, orders)
        return OpCounters(_acc(space, orders, None), pr * L * L, pr * (L + L * L), 0)
    return OpCounters(_acc(space, orders, None), 1, 0, 0)


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------
def _engine():
    from .engine import get_engine

    return get_engine()


def _weight_grid(emap: ElementMap, nodes: np.ndarray, mass_weight):
    """Mass weight sampled at the tensor nodes (gram.py:78-90): None for a
    constant, which is passed to the device as the per-element coefficient."""
    if mass_weight is None or np.isscalar(mass_weight):
        return None
    L = nodes.size
    grid = np.empty((L, L, L))
    for l in range(L):
        for m in range(L):
            for n in range(L):
                grid[l, m, n] = float(mass_weight(map_position(emap, (nodes[l], nodes[m], nodes[n]))))
    return grid


def _scalar(mass_weight) -> float:
    return 1.0 if mass_weight is None or not np.isscalar(mass_weight) else float(mass_weight)


def _device_matrix(sig: SpaceSignature, emap: ElementMap, path: str, L: int, coef: float,
                   wgrid=None, rule: Rule1D | None = None) -> np.ndarray:
    eng = _engine()
    N = dim(sig)
    nodes = weights = None
    if rule is not None:
        nodes, weights = rule.nodes, rule.weights
    packed, _ = eng.integrate(sig.space, path, sig.orders, L, np.array([emap.kind_code], np.int32),
                              emap.params.reshape(1, 24), np.array([coef]),
                              None if wgrid is None else wgrid.reshape(1, -1), nodes=nodes,
                              weights=weights)
    full = eng.expand(packed, N)
    return full[0].cpu().numpy()


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------
def gram_tensorized(sig: SpaceSignature, emap: ElementMap, rule1d: Rule1D | None = None,
                    loop_order: str = "standard", *, mass_weight=None) -> GramResult:
    """Sum-factorized Gram matrix (gram.py:139-158) on the GPU."""
    if loop_order not in ("standard", "alternative"):
        raise ValueError("loop_order must be 'standard' or 'alternative'")
    if rule1d is None:
        rule1d = gauss_rule(default_rule_order(sig.space, sig.orders))
    L = rule1d.nodes.size
    wgrid = _weight_grid(emap, rule1d.nodes, mass_weight)
    G = _device_matrix(sig, emap, "general", L, _scalar(mass_weight), wgrid, rule1d)
    return GramResult(G, counters(sig.space, sig.orders, "tensorized", L, loop_order))


def gram_simplified(sig: SpaceSignature, emap: ElementMap, ftab: FTable | None = None,
                    rule1d: Rule1D | None = None, *, mass_weight=None) -> GramResult:
    """Simplified Gram matrix (gram.py:161-205): constant-Jacobian maps on the
    closed-form O(p^6) kernel (path 1, simp_*_const), extrusion maps on the
    O(p^6) extrusion kernel (path 2, simp_*_ext: F tables in xi1, the 1D rule
    squared in (xi2, xi3) at xi1 = 0.5)."""
    klass = classify(emap)
    if klass == "general":
        raise SimplificationNotApplicableError(
            f"map kind {emap.kind!r} (class 'general') admits no simplification")
    if ftab is not None and ftab.p_max < max(sig.orders) + 1:
        raise ValueError("F table too small for the requested orders")
    if mass_weight is not None and not np.isscalar(mass_weight):
        raise ValueError("simplified backends support constant mass weights only")
    c = _scalar(mass_weight)
    if klass == "constant-jacobian":
        G = _device_matrix(sig, emap, "affine", 1, c)
        return GramResult(G, counters(sig.space, sig.orders, "simplified"))
    if rule1d is None:
        rule1d = gauss_rule(default_rule_order(sig.space, sig.orders))
    L = rule1d.nodes.size
    G = _device_matrix(sig, emap, "extrusion", L, c, None, rule1d)
    return GramResult(G, counters(sig.space, sig.orders, "simplified", L, klass="extrusion"))


def _rule3d_factor(rule3d: Rule3D) -> Rule1D:
    """The 1D factor of a tensor-product Rule3D (quadrature.py:69-83: points
    lexicographic in (l, m, n), weights w_l w_m w_n).  The Gauss tensor rule of
    its order returns gauss_rule(order) itself (bit-exact nodes/weights);
    any other tensor rule its extracted factor; a rule that is not a tensor
    product raises ValueError (the device kernels are sum-factorized)."""
    pts = np.asarray(rule3d.points, dtype=np.float64)
    wts = np.asarray(rule3d.weights, dtype=np.float64)
    n3 = wts.size
    L = int(round(n3 ** (1.0 / 3.0)))
    if L < 1 or L ** 3 != n3 or pts.shape != (n3, 3):
        raise ValueError("rule3d is not a tensor-product rule (L^3 points expected)")
    g = gauss_rule(L)
    nodes = pts[:L, 2].copy()
    w0 = np.cbrt(wts[0])
    weights = wts[:L] / (w0 * w0)
    cand = g if (np.array_equal(nodes, g.nodes) and np.allclose(weights, g.weights, rtol=1e-14, atol=0)) \
        else Rule1D(nodes=nodes, weights=weights, order=L)
    ll, mm, nn = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
    tp = np.stack([cand.nodes[ll.ravel()], cand.nodes[mm.ravel()], cand.nodes[nn.ravel()]], axis=1)
    tw = cand.weights[ll.ravel()] * cand.weights[mm.ravel()] * cand.weights[nn.ravel()]
    if not (np.array_equal(tp, pts) and np.allclose(tw, wts, rtol=1e-13, atol=0)):
        raise ValueError("rule3d is not a tensor-product rule; the device path integrates "
                         "with sum factorization over a 1D rule")
    return cand


def gram_conventional(sig: SpaceSignature, emap: ElementMap, rule3d: Rule3D | None = None, *,
                      mass_weight=None) -> GramResult:
    """Conventional-backend signature (gram.py:101-124).  The O(p^9) algorithm
    is out of scope; the matrix is the same tensor-rule integral computed by
    the sum-factorized device kernel with the rule's 1D factor
    (`_rule3d_factor`), and the counters are the conventional closed forms."""
    if rule3d is None:
        rule = gauss_rule(default_rule_order(sig.space, sig.orders))
    else:
        rule = _rule3d_factor(rule3d)
    L = rule.nodes.size
    wgrid = _weight_grid(emap, rule.nodes, mass_weight)
    G = _device_matrix(sig, emap, "general", L, _scalar(mass_weight), wgrid, rule)
    return GramResult(G, counters(sig.space, sig.orders, "conventional", L))


def gram(sig: SpaceSignature, emap: ElementMap, backend: str, *, rule_order: int | None = None,
         loop_order: str = "alternative", mass_weight=None) -> GramResult:
    """Dispatcher with a shared rule order (gram.py:208-232)."""
    L = rule_order if rule_order is not None else default_rule_order(sig.space, sig.orders)
    if backend == "conventional":
        from .quadrature import tensor_rule

        return gram_conventional(sig, emap, tensor_rule(L), mass_weight=mass_weight)
    if backend == "tensorized":
        return gram_tensorized(sig, emap, gauss_rule(L), loop_order, mass_weight=mass_weight)
    if backend == "simplified":
        return gram_simplified(sig, emap, None, gauss_rule(L), mass_weight=mass_weight)
    raise ValueError(f"unknown backend {backend!r}; choices: {BACKENDS}")


def gram_block(sig: SpaceSignature, emap: ElementMap, backend: str = "conventional",
               copies: int = 1, **kwargs) -> GramResult:
    """Block-diagonal replication for vector/matrix-valued spaces (gram.py:235-253)."""
    if copies not in (1, 3):
        raise ValueError("copies must be 1 or 3")
    base = gram(sig, emap, backend, **kwargs)
    if copies == 1:
        return base
    N = base.matrix.shape[0]
    M = np.zeros((3 * N, 3 * N))
    for c in range(3):
        M[c * N:(c + 1) * N, c * N:(c + 1) * N] = base.matrix
    return GramResult(M, base.counters)


def gram_batched(space: str, orders, kind, params, coef=None, *, path: str = "general",
                 rule_order: int | None = None, wgrid=None, out=None, stream=None, device=None,
                 rule: Rule1D | None = None, check_status: bool = True):
    """Batched native entry: E elements -> packed upper triangles.

    kind int32 [E], params float64 [E, 24], coef float64 [E] (mass-term
    weight, default 1), optional wgrid float64 [E, L^3]; torch tensors on the
    device or host arrays.  path: "general" (gram_tensorized), "affine"
    (constant-Jacobian gram_simplified) or "extrusion" (extrusion-map
    gram_simplified, rule_order points in xi2 and xi3).  `rule` (a Rule1D)
    replaces the Gauss rule of `rule_order` points.  Returns (packed
    [E, N(N+1)/2] float64 CUDA tensor, status [E] int32 CUDA tensor) --
    row-major upper triangles.  check_status=False skips the host read of the
    status word (no synchronisation; see GramEngine.raise_for_status)."""
    from .engine import get_engine

    sig = SpaceSignature(space, orders)
    L = rule_order if rule_order is not None else default_rule_order(space, sig.orders)
    nodes = weights = None
    if rule is not None:
        L = int(rule.nodes.size)
        nodes, weights = rule.nodes, rule.weights
    if path == "affine":
        L, nodes, weights = 1, None, None
    eng = get_engine(device)
    return eng.integrate(space, path, sig.orders, L, kind, params, coef, wgrid, out=out,
                         nodes=nodes, weights=weights, stream=stream, check_status=check_status)
