"""Element maps of the drop-in API.

Mirrors /root/reference/pkg/src/hexgram/geometry.py: the (kind, params[24])
encoding shared with the compiled kernels (KIND_CODES 46-52, constructors
83-119), the declared-kind classification (205-211) and the construction-time
orientation check (214-223).  Jacobians for batches are evaluated on the GPU
by the metric kernel; the host versions here serve single-element API calls
(eval_geometry, map_position for callable mass weights).
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import DegenerateMapError
from .quadrature import gauss_rule

KIND_CODES = {
    "identity": 0,
    "diagonal-affine": 1,
    "general-affine": 2,
    "extrusion": 3,
    "trilinear": 4,
}
KIND_NAMES = {v: k for k, v in KIND_CODES.items()}
N_PARAMS = 24
_CORNERS = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], dtype=float)


@dataclass(frozen=True)
class ElementMap:
    kind: str
    params: np.ndarray = field(default_factory=lambda: np.zeros(N_PARAMS))

    def __post_init__(self):
        if self.kind not in KIND_CODES:
            raise ValueError(f"unknown map kind {self.kind!r}")
        par = np.asarray(self.params, dtype=float)
        if par.shape != (N_PARAMS,):
            raise ValueError(f"params must have shape ({N_PARAMS},)")
        object.__setattr__(self, "params", par)
        _check_orientation(self)

    @property
    def kind_code(self) -> int:
        return KIND_CODES[self.kind]


@dataclass(frozen=True)
class JacobianData:
    J: np.ndarray
    Jinv: np.ndarray
    detJ: float
    D: np.ndarray
    C: np.ndarray


def identity_map() -> ElementMap:
    return ElementMap("identity", np.zeros(N_PARAMS))


def diagonal_affine_map(lams, shift=(0.0, 0.0, 0.0)) -> ElementMap:
    p = np.zeros(N_PARAMS)
    p[0:3], p[3:6] = lams, shift
    return ElementMap("diagonal-affine", p)


def general_affine_map(matrix, shift=(0.0, 0.0, 0.0)) -> ElementMap:
    p = np.zeros(N_PARAMS)
    p[0:9] = np.asarray(matrix, dtype=float).reshape(9)
    p[9:12] = shift
    return ElementMap("general-affine", p)


def extrusion_map(lam1: float, shift1: float, quad_vertices) -> ElementMap:
    p = np.zeros(N_PARAMS)
    p[0], p[1] = lam1, shift1
    p[2:10] = np.asarray(quad_vertices, dtype=float).reshape(8)
    return ElementMap("extrusion", p)


def trilinear_map(vertices) -> ElementMap:
    return ElementMap("trilinear", np.asarray(vertices, dtype=float).reshape(24).copy())


def jacobians(kind: str, params: np.ndarray, xi: np.ndarray) -> np.ndarray:
    """J[q, r, c] = d x_r / d xi_c at points xi[q] (vectorised over points)."""
    xi = np.atleast_2d(np.asarray(xi, dtype=float))
    n = xi.shape[0]
    p = params
    J = np.zeros((n, 3, 3))
    if kind == "identity":
        J[:] = np.eye(3)
    elif kind == "diagonal-affine":
        J[:] = np.diag(p[0:3])
    elif kind == "general-affine":
        J[:] = p[0:9].reshape(3, 3)
    elif kind == "extrusion":
        x2, x3 = xi[:, 1:2], xi[:, 2:3]
        v00, v10, v01, v11 = p[2:4], p[4:6], p[6:8], p[8:10]
        d2 = (v10 - v00) * (1.0 - x3) + (v11 - v01) * x3
        d3 = (v01 - v00) * (1.0 - x2) + (v11 - v10) * x2
        J[:, 0, 0] = p[0]
        J[:, 1:, 1] = d2
        J[:, 1:, 2] = d3
    else:
        v = p.reshape(8, 3)
        f = np.where(_CORNERS[None] == 1, xi[:, None, :], 1.0 - xi[:, None, :])  # (n, 8, 3)
        g = np.where(_CORNERS == 1, 1.0, -1.0)  # (8, 3)
        for d in range(3):
            others = [e for e in range(3) if e != d]
            coeff = g[None, :, d] * f[:, :, others[0]] * f[:, :, others[1]]  # (n, 8)
            J[:, :, d] = coeff @ v
    return J


def map_position(emap: ElementMap, xi) -> np.ndarray:
    x1, x2, x3 = (float(c) for c in xi)
    p = emap.params
    if emap.kind == "identity":
        return np.array([x1, x2, x3])
    if emap.kind == "diagonal-affine":
        return p[3:6] + p[0:3] * np.array([x1, x2, x3])
    if emap.kind == "general-affine":
        return p[9:12] + p[0:9].reshape(3, 3) @ np.array([x1, x2, x3])
    if emap.kind == "extrusion":
        v00, v10, v01, v11 = p[2:4], p[4:6], p[6:8], p[8:10]
        planar = (v00 * (1 - x2) * (1 - x3) + v10 * x2 * (1 - x3) + v01 * (1 - x2) * x3
                  + v11 * x2 * x3)
        return np.array([p[1] + p[0] * x1, planar[0], planar[1]])
    xi = np.array([x1, x2, x3])
    w = np.prod(np.where(_CORNERS == 1, xi, 1.0 - xi), axis=1)
    return w @ p.reshape(8, 3)


def eval_geometry(emap: ElementMap, xi) -> JacobianData:
    J = jacobians(emap.kind, emap.params, np.asarray(xi, dtype=float))[0]
    det = float(np.linalg.det(J))
    if det <= 0.0:
        raise DegenerateMapError(det, xi)
    Ji = np.linalg.inv(J)
    return JacobianData(J=J, Jinv=Ji, detJ=det, D=Ji @ Ji.T, C=J.T @ J)


def classify(emap: ElementMap) -> str:
    """Declared by kind, never inferred numerically (geometry.py:205-211)."""
    if emap.kind in ("identity", "diagonal-affine", "general-affine"):
        return "constant-jacobian"
    if emap.kind == "extrusion":
        return "extrusion"
    return "general"


_CHECK_PTS = None


def _check_orientation(emap: ElementMap) -> None:
    """det J > 0 at the 6-point tensor Gauss nodes (geometry.py:214-223)."""
    global _CHECK_PTS
    if _CHECK_PTS is None:
        n = gauss_rule(6).nodes
        _CHECK_PTS = np.stack(np.meshgrid(n, n, n, indexing="ij"), -1).reshape(-1, 3)
    det = np.linalg.det(jacobians(emap.kind, emap.params, _CHECK_PTS))
    bad = np.nonzero(det <= 0.0)[0]
    if bad.size:
        q = int(bad[0])
        raise DegenerateMapError(float(det[q]), tuple(_CHECK_PTS[q]))


_PRESETS = {
    "identity": identity_map,
    "diagonal-affine": lambda: diagonal_affine_map((2.0, 1.0, 1.0)),
    "general-affine": lambda: general_affine_map(
        [[1.0, 0.3, 0.1], [0.0, 1.1, 0.2], [0.05, 0.0, 0.9]], (0.2, -0.1, 0.4)),
    "extrusion": lambda: extrusion_map(1.0, 0.0, [
        (0.0, 0.0), (np.cos(np.pi / 6), np.sin(np.pi / 6)),
        (-np.sin(np.pi / 6), np.cos(np.pi / 6)),
        (np.cos(np.pi / 6) - np.sin(np.pi / 6) + 0.15, np.sin(np.pi / 6) + np.cos(np.pi / 6) + 0.1)]),
    "trilinear": lambda: trilinear_map([
        [0.0, 0.0, 0.0], [1.0, 0.0, 0.05], [0.0, 1.0, 0.0], [1.1, 1.05, 0.0],
        [0.0, 0.05, 1.0], [1.0, 0.0, 1.0], [-0.05, 0.9, 1.0], [1.1, 1.05, 0.95]]),
}
PRESET_MAP_NAMES = tuple(_PRESETS)


def preset_map(name: str) -> ElementMap:
    """The canonical map of each kind used by the reference's tests and CLI
    (geometry.py:268-312)."""
    try:
        return _PRESETS[name]()
    except KeyError:
        raise ValueError(f"unknown map preset {name!r}; choices: {PRESET_MAP_NAMES}")
