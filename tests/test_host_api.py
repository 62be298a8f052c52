"""Host-side objects of the drop-in API against the reference's golden vectors
and its documented behaviour (pkg/tests/test_quadrature.py, test_poly1d.py,
test_geometry.py, test_spaces.py patterns).  CPU only."""

import numpy as np
import pytest

import paper_1711_00984_b200 as hx
from paper_1711_00984_b200.geometry import jacobians


def test_gauss_rule_matches_reference(golden):
    for L in range(1, 17):
        r = hx.gauss_rule(L)
        np.testing.assert_allclose(r.nodes, golden[f"rule_{L}_nodes"], atol=2e-16, rtol=0)
        np.testing.assert_allclose(r.weights, golden[f"rule_{L}_weights"], atol=2e-16, rtol=0)
        assert abs(r.weights.sum() - 1.0) < 1e-14
    with pytest.raises(hx.InvalidOrderError):
        hx.gauss_rule(0)
    with pytest.raises(hx.InvalidOrderError):
        hx.gauss_rule(33)


def test_default_rule_order():
    assert hx.default_rule_order("L2", (3, 2, 4)) == 4
    assert hx.default_rule_order("Hcurl", (3, 2, 4)) == 5


def test_shape_tables_match_reference(golden):
    for k, x in enumerate(golden["shape_pts"]):
        t = hx.shape1_h1(12, float(x))
        np.testing.assert_allclose(t.chi, golden["shape_chi"][k], atol=1e-15, rtol=0)
        np.testing.assert_allclose(t.dchi, golden["shape_dchi"][k], atol=1e-15, rtol=0)
        np.testing.assert_allclose(hx.shape1_l2(12, float(x)), golden["shape_nu"][k], atol=1e-15)
    with pytest.raises(hx.DomainError):
        hx.shape1_h1(3, 1.5)


def test_ftable_matches_reference(golden):
    np.testing.assert_array_equal(hx.ftable(12).stacked, golden["ftable_12"])
    assert hx.f_entry(1, 0, 3, 2) == golden["ftable_12"][2, 3, 2]


def test_geometry_matches_reference(golden):
    names = {v: k for k, v in hx.geometry.KIND_CODES.items()}
    for i in range(golden["geo_kind"].shape[0]):
        kind = names[int(golden["geo_kind"][i])]
        J = jacobians(kind, golden["geo_params"][i], golden["geo_xi"][i])[0]
        np.testing.assert_allclose(J, golden["geo_J"][i], atol=1e-15, rtol=0)
        em = hx.ElementMap(kind, golden["geo_params"][i])
        g = hx.eval_geometry(em, golden["geo_xi"][i])
        np.testing.assert_allclose(g.detJ, golden["geo_det"][i], rtol=1e-14)
        np.testing.assert_allclose(g.C @ g.D, np.eye(3), atol=1e-13)


def test_degenerate_map_rejected():
    verts = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], float)
    verts[:, 0] = 1.0 - verts[:, 0]
    with pytest.raises(hx.DegenerateMapError):
        hx.trilinear_map(verts)


def test_classify_is_declared_by_kind():
    assert hx.classify(hx.preset_map("general-affine")) == "constant-jacobian"
    assert hx.classify(hx.preset_map("extrusion")) == "extrusion"
    assert hx.classify(hx.preset_map("trilinear")) == "general"


def test_flat_index_bijection():
    for space in ("H1", "Hcurl", "Hdiv", "L2"):
        sig = hx.SpaceSignature(space, (2, 3, 4))
        N = hx.dim(sig)
        seen = set()
        for I in range(N):
            a, ids = hx.flat_to_multi(sig, I)
            assert hx.multi_to_flat(sig, a, ids) == I
            seen.add((a, ids))
        assert len(seen) == N
    with pytest.raises(hx.InvalidOrderError):
        hx.SpaceSignature("H1", (0, 1, 1))
    with pytest.raises(ValueError):
        hx.SpaceSignature("H2", (1, 1, 1))


def test_simplified_rejects_before_device():
    sig = hx.SpaceSignature("L2", (2, 2, 2))
    with pytest.raises(hx.SimplificationNotApplicableError):
        hx.gram_simplified(sig, hx.preset_map("trilinear"))
    with pytest.raises(ValueError):
        hx.gram_simplified(sig, hx.identity_map(), mass_weight=lambda x: 1.0)
    with pytest.raises(ValueError):
        hx.gram_tensorized(sig, hx.identity_map(), loop_order="diagonal")
    with pytest.raises(ValueError):
        hx.gram(sig, hx.identity_map(), "magic")


def test_counters_closed_forms():
    c = hx.counters("L2", (4, 4, 4), "tensorized", 4, "standard")
    assert c.accumulations == 4 * (4 * 5 // 2) ** 3  # test_gram.py:114-118
    assert c.geometry_calls == 4 ** 3 * (4 * 5 // 2)  # test_gram.py:120-126
    a = hx.counters("L2", (4, 4, 4), "tensorized", 4, "alternative")
    assert a.geometry_calls == 4 ** 3
    assert hx.counters("L2", (3, 3, 3), "conventional", 3).accumulations == 3 ** 6 * (3 ** 3 + 1) // 2


def test_product_package_never_uses_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may touch oracle/."""
    import pathlib

    pkg = pathlib.Path(hx.__file__).parent
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "oracle" not in f.read_text().replace("CPU oracle", ""), f


def test_seeded_batches_are_valid_maps():
    from paper_1711_00984_b200.inputs import WORKLOADS

    for wl in WORKLOADS.values():
        b = wl.batch(8)
        for e in range(8):
            kind = "trilinear" if b.kind[e] == 4 else "general-affine"
            hx.ElementMap(kind, b.params[e])  # orientation check passes


def test_rule3d_factor():
    """gram_conventional's Rule3D handling (gram.py:101-124): the Gauss tensor
    rule maps back to gauss_rule(L) exactly, a non-Gauss tensor rule to its own
    1D factor, and a rule that is not a tensor product is rejected."""
    import numpy as np
    import pytest

    from paper_1711_00984_b200.gram import _rule3d_factor
    from paper_1711_00984_b200.quadrature import Rule3D, gauss_rule, tensor_rule

    for L in range(1, 12):
        r, g = _rule3d_factor(tensor_rule(L)), gauss_rule(L)
        np.testing.assert_array_equal(r.nodes, g.nodes)
        np.testing.assert_array_equal(r.weights, g.weights)
    n = np.array([0.1, 0.5, 0.8])
    w = np.array([0.3, 0.3, 0.4])
    pts = np.stack(np.meshgrid(n, n, n, indexing="ij"), -1).reshape(-1, 3)
    wts = np.einsum("i,j,k->ijk", w, w, w).ravel()
    r = _rule3d_factor(Rule3D(pts, wts, 3))
    np.testing.assert_array_equal(r.nodes, n)
    np.testing.assert_allclose(r.weights, w, rtol=1e-15)
    bad = pts.copy()
    bad[5, 0] = 0.33
    for P, W in ((bad, wts), (pts, wts * np.linspace(1, 1.1, 27)), (pts[:20], wts[:20])):
        with pytest.raises(ValueError):
            _rule3d_factor(Rule3D(P, W, 3))
