"""OpCounters of the drop-in API (all four fields) against the reference's own
counters for every backend and loop order (tests/golden/golden_counters.npz,
written by tests/golden/make_counters.py from /root/reference gram.py:101-232).

CPU only: the counters are closed forms (paper_1711_00984_b200/gram.py
`counters`), independent of the device computation."""

import os

import numpy as np

from paper_1711_00984_b200.gram import counters

HERE = os.path.dirname(os.path.abspath(__file__))
SPACES = ("H1", "Hcurl", "Hdiv", "L2")
MAPS = ("general-affine", "extrusion", "trilinear")


def _rows():
    return np.load(os.path.join(HERE, "golden", "golden_counters.npz"))["rows"]


def test_counter_fixture_covers_every_backend():
    rows = _rows()
    assert set(rows[:, 1]) == {0, 1, 2, 3}
    assert set(rows[:, 0]) == {0, 1, 2, 3}


def test_counters_match_reference_all_fields():
    bad = []
    for r in _rows():
        si, bi, mi, p1, p2, p3, L = (int(x) for x in r[:7])
        want = tuple(int(x) for x in r[7:])
        space, orders = SPACES[si], (p1, p2, p3)
        if bi == 0:
            c = counters(space, orders, "conventional", L)
        elif bi in (1, 2):
            c = counters(space, orders, "tensorized", L, "standard" if bi == 1 else "alternative")
        else:
            klass = "extrusion" if MAPS[mi] == "extrusion" else "constant-jacobian"
            c = counters(space, orders, "simplified", L, klass=klass)
        got = (c.accumulations, c.geometry_calls, c.shape1_calls, c.shape3_calls)
        if got != want:
            bad.append((space, orders, bi, MAPS[mi], L, got, want))
    assert not bad, bad[:5]
