"""Host-side 1D polynomial tables of the drop-in API.

Mirrors the public surface of /root/reference/pkg/src/hexgram/poly1d.py
(legendre_all 62-74, shape1_h1 77-92, shape1_l2 95-99, FTable/ftable
228-266).  The device path generates the same tables on the GPU
(hxg_make_tables); `ftable` is accepted by gram_simplified for signature
compatibility and range checking.
"""

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import DomainError, InvalidOrderError

DEFAULT_P_MAX = 12


@dataclass(frozen=True)
class LegendreEval:
    values: np.ndarray
    point: float


@dataclass(frozen=True)
class ShapeTable1D:
    chi: np.ndarray
    dchi: np.ndarray
    point: float


def _legendre(n: int, xi: float) -> np.ndarray:
    t = 2.0 * xi - 1.0
    v = np.empty(n + 1)
    v[0] = 1.0
    if n >= 1:
        v[1] = t
    for i in range(2, n + 1):
        v[i] = ((2 * i - 1) * t * v[i - 1] - (i - 1) * v[i - 2]) / i
    return v


def _check(xi: float) -> None:
    if not 0.0 <= xi <= 1.0:
        raise DomainError(f"evaluation point {xi} outside the master interval [0, 1]")


def legendre_all(n: int, xi: float) -> LegendreEval:
    if n < 0:
        raise InvalidOrderError("legendre_all requires n >= 0")
    _check(xi)
    return LegendreEval(_legendre(n, xi), xi)


def shape1_h1(p: int, xi: float) -> ShapeTable1D:
    """chi_0 = 1 - xi, chi_1 = xi, chi_i = (P_i - P_{i-2}) / (2 (2i - 1)); chi'_i = P_{i-1}."""
    if p < 1:
        raise InvalidOrderError("shape1_h1 requires p >= 1")
    _check(xi)
    P = _legendre(p, xi)
    chi = np.empty(p + 1)
    dchi = np.empty(p + 1)
    chi[:2] = (1.0 - xi, xi)
    dchi[:2] = (-1.0, 1.0)
    i = np.arange(2, p + 1)
    chi[2:] = (P[2:] - P[:-2]) / (2.0 * (2 * i - 1))
    dchi[2:] = P[1:-1]
    return ShapeTable1D(chi, dchi, xi)


def shape1_l2(p: int, xi: float) -> np.ndarray:
    if p < 1:
        raise InvalidOrderError("shape1_l2 requires p >= 1")
    _check(xi)
    return _legendre(p - 1, xi)


def _f00(i: int, j: int) -> float:
    hi, lo = max(i, j), min(i, j)
    if lo >= 2:
        if hi == lo:
            return (1.0 / (2 * lo + 1) + 1.0 / (2 * lo - 3)) / (4.0 * (2 * lo - 1) ** 2)
        if hi == lo + 2:
            return -1.0 / (4.0 * (2 * lo + 3) * (2 * lo - 1) * (2 * lo + 1))
        return 0.0
    table = {(0, 0): 1 / 3, (1, 0): 1 / 6, (2, 0): -1 / 12, (3, 0): 1 / 60,
             (1, 1): 1 / 3, (2, 1): -1 / 12, (3, 1): -1 / 60}
    return table.get((hi, lo), 0.0)


def _f01(i: int, j: int) -> float:
    if j == 0:
        return -_f01(i, 1)
    small = {(0, 1): 0.5, (0, 2): -1 / 6, (1, 1): 0.5, (1, 2): 1 / 6, (2, 1): -1 / 6, (2, 3): 1 / 30}
    if i <= 2:
        return small.get((i, j), 0.0)
    if j == i + 1:
        return 1.0 / (2.0 * (2 * i - 1) * (2 * i + 1))
    if j == i - 1:
        return -1.0 / (2.0 * (2 * i - 1) * (2 * i - 3))
    return 0.0


def _f11(i: int, j: int) -> float:
    hi, lo = max(i, j), min(i, j)
    if lo >= 1:
        return 1.0 / (2 * hi - 1) if hi == lo else 0.0
    return {0: 1.0, 1: -1.0}.get(hi, 0.0)


def f_entry(r: int, s: int, i: int, j: int) -> float:
    if r not in (0, 1) or s not in (0, 1):
        raise ValueError("derivative flags r, s must be 0 or 1")
    if i < 0 or j < 0:
        raise ValueError("shape indices must be non-negative")
    if (r, s) == (0, 0):
        return _f00(i, j)
    if (r, s) == (0, 1):
        return _f01(i, j)
    if (r, s) == (1, 0):
        return _f01(j, i)
    return _f11(i, j)


@dataclass(frozen=True)
class FTable:
    p_max: int
    f00: np.ndarray
    f01: np.ndarray
    f11: np.ndarray
    stacked: np.ndarray

    def entry(self, r: int, s: int, i: int, j: int) -> float:
        if not (0 <= i <= self.p_max and 0 <= j <= self.p_max):
            raise ValueError(f"indices ({i}, {j}) exceed table p_max = {self.p_max}")
        return float(self.stacked[2 * r + s, i, j])


@lru_cache(maxsize=None)
def ftable(p_max: int = DEFAULT_P_MAX) -> FTable:
    if p_max < 1:
        raise InvalidOrderError("ftable requires p_max >= 1")
    n = p_max + 1
    f00 = np.array([[_f00(i, j) for j in range(n)] for i in range(n)])
    f01 = np.array([[_f01(i, j) for j in range(n)] for i in range(n)])
    f11 = np.array([[_f11(i, j) for j in range(n)] for i in range(n)])
    stacked = np.ascontiguousarray(np.stack([f00, f01, f01.T, f11]))
    return FTable(p_max, f00, f01, f11, stacked)
