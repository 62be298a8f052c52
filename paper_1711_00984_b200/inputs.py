"""Seeded synthetic element batches for the BASELINE.json configs.

The reference publishes no dataset; the paper times a single master
hexahedron.  The batches below are the canonical generator of
SURVEY.md section 8(d): the same ``kind[E]``, ``params[E, 24]`` and
``coef[E]`` arrays feed the CUDA path, the CPU oracle and the reference
(parameter layouts of /root/reference/pkg/src/hexgram/geometry.py:45-119).

Draw order is fixed here once:
* trilinear (kind 4): verts = CUBE + U(-0.1, 0.1)^(E, 8, 3); then coef.
* affine (kind 2):    A = I + U(-0.2, 0.2)^(E, 3, 3); shift = U(0, 1)^(E, 3);
  then coef.
coef ~ U(0.5, 2) when the config asks for a variable coefficient, else 1.
"""

from dataclasses import dataclass

import numpy as np

KIND_CODES = {
    "identity": 0,
    "diagonal-affine": 1,
    "general-affine": 2,
    "extrusion": 3,
    "trilinear": 4,
}

# geometry.py:115-119: vertex k is the image of corner (k&1, k>>1&1, k>>2&1)
CUBE = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], dtype=np.float64)


@dataclass(frozen=True)
class ElementBatch:
    kind: np.ndarray  # int32 [E]
    params: np.ndarray  # float64 [E, 24]
    coef: np.ndarray  # float64 [E]

    @property
    def size(self) -> int:
        return int(self.kind.shape[0])

    def slice(self, lo: int, hi: int) -> "ElementBatch":
        return ElementBatch(self.kind[lo:hi], self.params[lo:hi], self.coef[lo:hi])


def trilinear_batch(E: int, seed: int, perturb: float = 0.1, variable_coef: bool = False):
    rng = np.random.default_rng(seed)
    verts = CUBE[None] + rng.uniform(-perturb, perturb, (E, 8, 3))
    params = np.ascontiguousarray(verts.reshape(E, 24))
    coef = rng.uniform(0.5, 2.0, E) if variable_coef else np.ones(E)
    return ElementBatch(np.full(E, 4, np.int32), params, np.ascontiguousarray(coef))


def affine_batch(E: int, seed: int, spread: float = 0.2, variable_coef: bool = False):
    rng = np.random.default_rng(seed)
    A = np.eye(3)[None] + rng.uniform(-spread, spread, (E, 3, 3))
    shift = rng.uniform(0.0, 1.0, (E, 3))
    params = np.zeros((E, 24))
    params[:, 0:9] = A.reshape(E, 9)
    params[:, 9:12] = shift
    coef = rng.uniform(0.5, 2.0, E) if variable_coef else np.ones(E)
    return ElementBatch(np.full(E, 2, np.int32), params, np.ascontiguousarray(coef))


def extrusion_batch(E: int, seed: int, spread: float = 0.1, variable_coef: bool = False):
    """Extrusion maps (kind 3, geometry.py:100-111): x1 = lam1 xi1 + shift1 with
    lam1 = 1 + U(-0.2, 0.2), shift1 = U(0, 1), and the planar quad
    (v00, v10, v01, v11) = unit-square corners + U(-spread, spread)^(4, 2)."""
    rng = np.random.default_rng(seed)
    lam1 = 1.0 + rng.uniform(-0.2, 0.2, E)
    shift1 = rng.uniform(0.0, 1.0, E)
    quad = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    verts = quad[None] + rng.uniform(-spread, spread, (E, 4, 2))
    params = np.zeros((E, 24))
    params[:, 0] = lam1
    params[:, 1] = shift1
    params[:, 2:10] = verts.reshape(E, 8)
    coef = rng.uniform(0.5, 2.0, E) if variable_coef else np.ones(E)
    return ElementBatch(np.full(E, 3, np.int32), params, np.ascontiguousarray(coef))


@dataclass(frozen=True)
class Workload:
    name: str
    space: str
    p: int
    L: int
    path: str  # "general" (O(p^7)), "affine" or "extrusion" (O(p^6))
    E: int
    seed: int
    maps: str  # "trilinear" | "affine" | "extrusion"
    variable_coef: bool = False

    @property
    def orders(self):
        return (self.p, self.p, self.p)

    def batch(self, E: int | None = None) -> ElementBatch:
        E = self.E if E is None else E
        if self.maps == "trilinear":
            return trilinear_batch(E, self.seed, variable_coef=self.variable_coef)
        if self.maps == "extrusion":
            return extrusion_batch(E, self.seed, variable_coef=self.variable_coef)
        return affine_batch(E, self.seed, variable_coef=self.variable_coef)


# BASELINE.json configs (L = p_test + 1 for every space, including L2).
WORKLOADS = {
    "c1_h1_p3_affine": Workload("c1_h1_p3_affine", "H1", 3, 4, "affine", 64, 0, "affine"),
    "c2_h1_p5_general": Workload("c2_h1_p5_general", "H1", 5, 6, "general", 4096, 1,
                                 "trilinear", True),
    "c3_hcurl_p6_general": Workload("c3_hcurl_p6_general", "Hcurl", 6, 7, "general", 2048, 2,
                                    "trilinear"),
    "c3_hcurl_p6_affine": Workload("c3_hcurl_p6_affine", "Hcurl", 6, 7, "affine", 2048, 2,
                                   "affine"),
    "c4_hdiv_p7_general": Workload("c4_hdiv_p7_general", "Hdiv", 7, 8, "general", 1024, 3,
                                   "trilinear"),
    "c4_l2_p7_general": Workload("c4_l2_p7_general", "L2", 7, 8, "general", 1024, 3,
                                 "trilinear"),
}


def dim(space: str, orders) -> int:
    """spaces.py:67-80."""
    p1, p2, p3 = orders
    if space == "H1":
        return (p1 + 1) * (p2 + 1) * (p3 + 1)
    if space == "L2":
        return p1 * p2 * p3
    if space == "Hdiv":
        return (p1 + 1) * p2 * p3 + p1 * (p2 + 1) * p3 + p1 * p2 * (p3 + 1)
    if space == "Hcurl":
        return p1 * (p2 + 1) * (p3 + 1) + (p1 + 1) * p2 * (p3 + 1) + (p1 + 1) * (p2 + 1) * p3
    raise ValueError(space)


def packed_size(space: str, orders) -> int:
    N = dim(space, orders)
    return N * (N + 1) // 2


def sweep_elements(space: str, p: int, budget_bytes: float = 100e9) -> int:
    """Config 5: E_p = floor(budget / B(p)), B = 8 N(N+1)/2."""
    return int(budget_bytes // (8 * packed_size(space, (p, p, p))))


# order-sweep points (BASELINE config 5), addressable by name for profiling
SWEEP_WORKLOADS = {
    f"c5_{sp.lower()}_p{p}_{path}": Workload(f"c5_{sp.lower()}_p{p}_{path}", sp, p, p + 1, path,
                                             sweep_elements(sp, p), 4, maps)
    for sp in ("H1", "Hcurl", "Hdiv") for p in range(2, 11)
    for path, maps in (("general", "trilinear"), ("affine", "affine"))
}
# extrusion-map simplified path (not a BASELINE config):
# the config-3 shape on extrusion maps, and the order sweep of config 5
EXTRUSION_WORKLOADS = {
    "x_hcurl_p6_extrusion": Workload("x_hcurl_p6_extrusion", "Hcurl", 6, 7, "extrusion", 2048, 5,
                                     "extrusion"),
    **{f"x5_{sp.lower()}_p{p}_extrusion": Workload(f"x5_{sp.lower()}_p{p}_extrusion", sp, p, p + 1,
                                                    "extrusion", sweep_elements(sp, p), 4, "extrusion")
       for sp in ("H1", "Hcurl", "Hdiv") for p in range(2, 11)},
}
ALL_WORKLOADS = {**WORKLOADS, **SWEEP_WORKLOADS, **EXTRUSION_WORKLOADS}
