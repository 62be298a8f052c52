"""Space signatures and index conventions of the drop-in API.

Mirrors /root/reference/pkg/src/hexgram/spaces.py (SpaceSignature 39-49,
dim 67-80, per-component digit ranges 95-102, flat <-> multi index 105-158).
The flat index defines the row/column order of every Gram matrix the
library writes.
"""

from dataclasses import dataclass

from .errors import InvalidOrderError

SPACES = ("H1", "Hcurl", "Hdiv", "L2")


@dataclass(frozen=True)
class SpaceSignature:
    space: str
    orders: tuple

    def __post_init__(self):
        if self.space not in SPACES:
            raise ValueError(f"unknown space {self.space!r}")
        orders = tuple(int(p) for p in self.orders)
        object.__setattr__(self, "orders", orders)
        if len(orders) != 3 or min(orders) < 1:
            raise InvalidOrderError("orders must be three positive integers")


def component_extents(space: str, a, orders):
    """Digit counts (n1, n2, n3) of component a (1-based) or of a scalar space."""
    if space == "H1":
        return tuple(p + 1 for p in orders)
    if space == "L2":
        return tuple(orders)
    if space == "Hdiv":
        return tuple(p + 1 if d == a else p for d, p in enumerate(orders, start=1))
    return tuple(p if d == a else p + 1 for d, p in enumerate(orders, start=1))


def _blocks(sig: SpaceSignature):
    if sig.space in ("H1", "L2"):
        return [component_extents(sig.space, None, sig.orders)]
    return [component_extents(sig.space, a, sig.orders) for a in (1, 2, 3)]


def dim(sig: SpaceSignature) -> int:
    return sum(n1 * n2 * n3 for n1, n2, n3 in _blocks(sig))


def multi_to_flat(sig: SpaceSignature, a, ids) -> int:
    vector = sig.space in ("Hdiv", "Hcurl")
    if vector and a not in (1, 2, 3):
        raise ValueError("vector spaces need component a in {1, 2, 3}")
    blocks = _blocks(sig)
    k = (a - 1) if vector else 0
    n1, n2, n3 = blocks[k]
    i1, i2, i3 = ids
    if not (0 <= i1 < n1 and 0 <= i2 < n2 and 0 <= i3 < n3):
        raise IndexError(f"digits {ids} out of range")
    off = sum(x * y * z for x, y, z in blocks[:k])
    return off + i1 + n1 * (i2 + n2 * i3)


def flat_to_multi(sig: SpaceSignature, I: int):
    N = dim(sig)
    if not 0 <= I < N:
        raise IndexError(f"flat index {I} out of range [0, {N})")
    vector = sig.space in ("Hdiv", "Hcurl")
    for k, (n1, n2, n3) in enumerate(_blocks(sig)):
        size = n1 * n2 * n3
        if I < size:
            ids = (I % n1, (I // n1) % n2, I // (n1 * n2))
            return (k + 1 if vector else None), ids
        I -= size
    raise AssertionError("unreachable")
