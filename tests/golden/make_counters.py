"""Golden OpCounters (all four fields) of the reference, for every backend and
loop order the drop-in reports counters for.

Run in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_counters.py

Writes tests/golden/golden_counters.npz: rows of
(space, backend, loop_order, map, p1, p2, p3, L, accumulations, geometry_calls,
shape1_calls, shape3_calls) produced by the reference's public API
(/root/reference/pkg/src/hexgram/gram.py:101-232).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import hexgram as hg  # noqa: E402
from hexgram.geometry import preset_map  # noqa: E402

OUT = os.path.join(HERE, "golden_counters.npz")
SPACES = ("H1", "Hcurl", "Hdiv", "L2")
# backend codes: 0 conventional, 1 tensorized std, 2 tensorized alt, 3 simplified
MAPS = ("general-affine", "extrusion", "trilinear")


def main():
    rows = []
    for si, space in enumerate(SPACES):
        for orders in [(1, 1, 1), (2, 3, 2), (3, 3, 3), (2, 3, 4), (4, 2, 1)]:
            sig = hg.SpaceSignature(space, orders)
            Ld = hg.default_rule_order(space, orders)
            for L in (Ld, Ld + 1):
                for mi, mname in enumerate(MAPS):
                    em = preset_map(mname)
                    if mname == "trilinear":
                        for bi, lo in ((1, "standard"), (2, "alternative")):
                            c = hg.gram(sig, em, "tensorized", rule_order=L, loop_order=lo).counters
                            rows.append([si, bi, mi, *orders, L, c.accumulations, c.geometry_calls,
                                         c.shape1_calls, c.shape3_calls])
                        if max(orders) <= 3:
                            c = hg.gram(sig, em, "conventional", rule_order=L).counters
                            rows.append([si, 0, mi, *orders, L, c.accumulations, c.geometry_calls,
                                         c.shape1_calls, c.shape3_calls])
                    else:
                        c = hg.gram(sig, em, "simplified", rule_order=L).counters
                        rows.append([si, 3, mi, *orders, L, c.accumulations, c.geometry_calls,
                                     c.shape1_calls, c.shape3_calls])
    np.savez_compressed(OUT, rows=np.array(rows, dtype=np.int64))
    print(f"wrote {len(rows)} counter rows to {OUT}")


if __name__ == "__main__":
    main()
