"""Parity of the sm_100a kernels (through the C ABI) with the CPU oracle and
the reference's golden vectors.  Tolerance: relative Frobenius error per
element matrix <= 1e-12 (BASELINE.json north_star), fp64."""

import numpy as np
import pytest

from conftest import golden_cases

pytestmark = pytest.mark.gpu

TOL = 1e-12
SPACES = ("H1", "Hcurl", "Hdiv", "L2")


def rel_fro(got_packed, ref_packed, N, orc):
    G = orc.unpack(got_packed, N)
    R = orc.unpack(ref_packed, N)
    return np.linalg.norm(G - R) / np.linalg.norm(R)


def check_batch(space, path, orders, L, b, orc, rule_order=None):
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim

    packed, status = gram_batched(space, orders, b.kind, b.params, b.coef, path=path,
                                  rule_order=L)
    torch.cuda.synchronize()
    got = packed.cpu().numpy()
    ref = orc.gram_batched(space, path, orders, L, b.kind, b.params, b.coef)
    N = dim(space, orders)
    worst = max(rel_fro(got[e], ref[e], N, orc) for e in range(b.size))
    assert worst <= TOL, (space, path, orders, L, worst)
    assert int(status.abs().sum()) == 0
    return worst


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("orders", [(1, 1, 1), (2, 2, 2), (2, 3, 2), (1, 2, 3), (3, 2, 3),
                                    (2, 3, 4), (4, 4, 4)])
def test_general_vs_oracle(space, orders, orc):
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(5, 100 + sum(orders), variable_coef=True)
    check_batch(space, "general", orders, max(orders) + 1, b, orc)


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("orders", [(1, 1, 1), (2, 2, 2), (3, 2, 3), (1, 2, 3), (4, 4, 4)])
def test_affine_vs_oracle(space, orders, orc):
    from paper_1711_00984_b200.inputs import affine_batch

    b = affine_batch(5, 200 + sum(orders), variable_coef=True)
    check_batch(space, "affine", orders, 1, b, orc)


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [3, 5, 6, 7, 8, 9, 10])
def test_high_order_general(space, p, orc):
    """Sweep orders (config 5): includes L > 8 (second kernel instantiation)
    and n1 > 8 (two DMMA row tiles)."""
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(2, 300 + p)
    check_batch(space, "general", (p, p, p), p + 1, b, orc)


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [6, 8, 10, 12])
def test_high_order_affine(space, p, orc):
    from paper_1711_00984_b200.inputs import affine_batch

    b = affine_batch(3, 400 + p)
    check_batch(space, "affine", (p, p, p), 1, b, orc)


def test_golden_cases_dropin_api(golden):
    """The reference's own matrices through the drop-in per-element API."""
    import paper_1711_00984_b200 as hx

    for c in golden_cases(golden):
        sig = hx.SpaceSignature(c["space"], c["orders"])
        kind_name = {0: "identity", 1: "diagonal-affine", 2: "general-affine", 3: "extrusion",
                     4: "trilinear"}[c["kind"]]
        em = hx.ElementMap(kind_name, c["params"])
        if c["path"] in ("affine", "extrusion"):
            res = hx.gram_simplified(sig, em, mass_weight=c["coef"])
        elif c["wgrid"] is not None:
            w = lambda x: 1.0 + x[0] ** 2 + 0.5 * x[1]  # noqa: E731 (make_golden.py)
            res = hx.gram_tensorized(sig, em, hx.gauss_rule(c["L"]), "alternative",
                                     mass_weight=w)
        else:
            res = hx.gram_tensorized(sig, em, hx.gauss_rule(c["L"]), "alternative",
                                     mass_weight=c["coef"])
        N = res.matrix.shape[0]
        R = np.zeros((N, N))
        iu = np.triu_indices(N)
        R[iu] = c["packed"]
        R.T[iu] = c["packed"]
        rel = np.linalg.norm(res.matrix - R) / np.linalg.norm(R)
        assert rel <= TOL, (c["space"], c["path"], c["orders"], kind_name, rel)
        np.testing.assert_array_equal(res.matrix, res.matrix.T)
        assert res.counters.accumulations == c["acc"]


@pytest.mark.parametrize("name", ["c1_h1_p3_affine", "c2_h1_p5_general", "c3_hcurl_p6_general",
                                  "c3_hcurl_p6_affine", "c4_hdiv_p7_general", "c4_l2_p7_general"])
def test_config_golden_samples(golden, name):
    """BASELINE config batches against the reference's own sampled entries."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import WORKLOADS

    wl = WORKLOADS[name]
    nel = 8 if name == "c1_h1_p3_affine" else 1
    b = wl.batch(max(nel, 4))
    packed, _ = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef, path=wl.path,
                             rule_order=wl.L)
    torch.cuda.synchronize()
    got = packed.cpu().numpy()
    for e in range(nel):
        pre = f"{name}_e{e}"
        if pre + "_packed" in golden.files:
            ref = golden[pre + "_packed"]
            vals, gv = ref, got[e]
        else:
            vals, gv = golden[pre + "_val"], got[e][golden[pre + "_idx"]]
        fro = golden[pre + "_fro"][0]
        assert np.linalg.norm(gv - vals) <= TOL * fro


def test_full_config_batches(orc):
    """Full BASELINE batch sizes: every element checked against the oracle on
    a strided sample, plus size-independent properties on all elements
    (finite, diagonal > 0)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import WORKLOADS, dim

    for name, wl in WORKLOADS.items():
        b = wl.batch()
        packed, status = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef,
                                      path=wl.path, rule_order=wl.L)
        torch.cuda.synchronize()
        assert int(status.abs().sum()) == 0
        N = dim(wl.space, wl.orders)
        assert bool(torch.isfinite(packed).all())
        diag_idx = torch.tensor([r * N - r * (r - 1) // 2 for r in range(N)], device=packed.device)
        assert bool((packed[:, diag_idx] > 0).all())
        sample = sorted(set([0, b.size - 1] + list(range(0, b.size, max(1, b.size // 6)))))[:8]
        ref = orc.gram_batched(wl.space, wl.path, wl.orders, wl.L, b.kind[sample],
                               b.params[sample], b.coef[sample])
        got = packed[sample].cpu().numpy()
        for k in range(len(sample)):
            assert rel_fro(got[k], ref[k], N, orc) <= TOL, (name, sample[k])
        del packed


def test_general_equals_affine_on_affine_maps():
    """Cross-path consistency (test_gram.py:145-153 pattern): on constant-
    Jacobian maps the O(p^7) and O(p^6) kernels agree to 1e-12."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import affine_batch

    for space in SPACES:
        for p in (3, 6):
            b = affine_batch(16, 500 + p, variable_coef=True)
            g, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, path="general",
                                rule_order=p + 1)
            a, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, path="affine")
            torch.cuda.synchronize()
            num = torch.linalg.norm(g - a, dim=1)
            den = torch.linalg.norm(a, dim=1)
            assert float((num / den).max()) <= TOL, (space, p)


def test_mass_weight_linearity():
    """The coefficient multiplies only the mass term (test_gram.py:231-238)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(4, 600)
    for space in SPACES:
        c0 = np.zeros(4)
        c1 = np.ones(4)
        c3 = np.full(4, 3.0)
        g0, _ = gram_batched(space, (3, 3, 3), b.kind, b.params, c0)
        g1, _ = gram_batched(space, (3, 3, 3), b.kind, b.params, c1)
        g3, _ = gram_batched(space, (3, 3, 3), b.kind, b.params, c3)
        torch.cuda.synchronize()
        lhs = g3 - g0
        rhs = 3.0 * (g1 - g0)
        assert float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(g1)) <= 1e-13


def test_edge_cases():
    import torch

    import paper_1711_00984_b200 as hx
    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    # empty batch
    b = trilinear_batch(1, 1)
    out, st = gram_batched("H1", (2, 2, 2), b.kind[:0], b.params[:0], b.coef[:0])
    assert out.shape == (0, 27 * 28 // 2)
    # unsupported order -> InvalidOrderError
    with pytest.raises(hx.InvalidOrderError):
        gram_batched("H1", (13, 2, 2), b.kind, b.params, b.coef)
    # trilinear kind on the affine path -> SimplificationNotApplicableError
    with pytest.raises(hx.SimplificationNotApplicableError):
        gram_batched("H1", (2, 2, 2), b.kind, b.params, b.coef, path="affine")
    with pytest.raises(hx.SimplificationNotApplicableError):
        hx.gram_simplified(hx.SpaceSignature("L2", (2, 2, 2)), hx.preset_map("trilinear"))
    # inverted element -> DegenerateMapError from the device status word
    par = b.params.copy().reshape(1, 8, 3)
    par[0, :, 0] = 1.0 - par[0, :, 0]  # mirror x: det < 0 everywhere
    with pytest.raises(hx.DegenerateMapError):
        gram_batched("H1", (2, 2, 2), b.kind, par.reshape(1, 24), b.coef)
    # L2 with the reference's default rule (L = max p) and loop-order counters
    sig = hx.SpaceSignature("L2", (3, 3, 3))
    r_std = hx.gram_tensorized(sig, hx.preset_map("trilinear"))
    r_alt = hx.gram_tensorized(sig, hx.preset_map("trilinear"), loop_order="alternative")
    np.testing.assert_array_equal(r_std.matrix, r_alt.matrix)
    assert r_std.counters.geometry_calls > r_alt.counters.geometry_calls
    torch.cuda.synchronize()


def test_host_entry_matches_device_entry():
    """hxg_gram_batched_host (host buffers, chunked, overlapped D2H) equals
    the device entry."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.engine import get_engine
    from paper_1711_00984_b200.inputs import packed_size, trilinear_batch

    b = trilinear_batch(40, 700, variable_coef=True)
    d, _ = gram_batched("Hcurl", (4, 4, 4), b.kind, b.params, b.coef)
    out = torch.empty((40, packed_size("Hcurl", (4, 4, 4))), dtype=torch.float64).pin_memory()
    status = np.zeros(40, np.int32)
    get_engine().integrate_host("Hcurl", "general", (4, 4, 4), 5, b.kind, b.params, b.coef,
                                out, status)
    np.testing.assert_array_equal(out.numpy(), d.cpu().numpy())
    assert status.sum() == 0


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10])
def test_specialized_equals_generic(space, p, monkeypatch):
    """The compile-time specialized kernel (isotropic p, L = p + 1) and the
    runtime-generic kernel agree to 1e-12 on the same batch."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(3, 800 + p, variable_coef=True)
    spec, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef)
    monkeypatch.setenv("HXG_FORCE_V2", "1")  # CTA-chunked specialization instead of warp units
    spec2, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef)
    monkeypatch.setenv("HXG_FORCE_GENERIC", "1")
    gen, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef)
    torch.cuda.synchronize()
    for got in (spec, spec2):
        rel = torch.linalg.norm(got - gen, dim=1) / torch.linalg.norm(gen, dim=1)
        assert float(rel.max()) <= TOL


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [1, 3, 5, 6, 8])
def test_affine_row_group_split_invariant(space, p, monkeypatch, orc):
    """The constant-Jacobian kernel gives bit-identical packed rows whether a CTA
    owns one row group, a few, or the whole element (HXG_AFF_RG overrides the
    size-based choice of aff_row_groups), and matches the oracle."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import affine_batch

    b = affine_batch(5, 900 + p, variable_coef=True)
    outs = []
    for rg in ("1", "3", "1000"):
        monkeypatch.setenv("HXG_AFF_RG", rg)
        got, st = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, path="affine")
        torch.cuda.synchronize()
        assert int(st.abs().sum()) == 0
        outs.append(got.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    ref = orc.gram_batched(space, "affine", (p, p, p), 1, b.kind, b.params, b.coef)
    rel = np.linalg.norm(outs[0] - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() <= TOL


# ---------------------------------------------------------------------------
# simplified extrusion path (path 2, simp_*_ext, _kernels.py:1405-1764)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("orders", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (2, 3, 2), (1, 2, 3), (4, 4, 4),
                                    (5, 5, 5), (6, 6, 6), (7, 7, 7), (8, 8, 8), (10, 10, 10)])
def test_extrusion_vs_oracle(space, orders, orc):
    """Extrusion maps through the C ABI (specialized kernel for isotropic p <= 10,
    the general kernels for anisotropic orders) against the C restatement of
    simp_*_ext, at the reference's default rule (L = p + 1, L2: p)."""
    from paper_1711_00984_b200.inputs import extrusion_batch
    from paper_1711_00984_b200.quadrature import default_rule_order

    b = extrusion_batch(4 if max(orders) < 8 else 2, 600 + sum(orders), variable_coef=True)
    check_batch(space, "extrusion", orders, default_rule_order(space, orders), b, orc)


@pytest.mark.parametrize("space", SPACES)
def test_extrusion_rule_orders(space, orc):
    """Rules other than the default (gram(..., rule_order=L)) on the extrusion path."""
    from paper_1711_00984_b200.inputs import extrusion_batch

    b = extrusion_batch(3, 650, variable_coef=True)
    for L in (2, 5, 9, 16):
        check_batch(space, "extrusion", (4, 4, 4), L, b, orc)


def test_extrusion_equals_general_on_extrusion_maps():
    """Same integral on two algorithms: the xi1 rule of the general path with
    L = p + 1 is exact for an xi1-independent Jacobian."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import extrusion_batch

    for space in SPACES:
        for p in (2, 5, 7):
            b = extrusion_batch(8, 700 + p, variable_coef=True)
            x, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, path="extrusion",
                                rule_order=p + 1)
            g, _ = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, rule_order=p + 1)
            torch.cuda.synchronize()
            rel = torch.linalg.norm(x - g, dim=1) / torch.linalg.norm(g, dim=1)
            assert float(rel.max()) <= TOL, (space, p, float(rel.max()))


def test_extrusion_path_rejects_trilinear_maps():
    import paper_1711_00984_b200 as hx
    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import extrusion_batch, trilinear_batch

    b = trilinear_batch(2, 5)
    with pytest.raises(hx.SimplificationNotApplicableError):
        gram_batched("H1", (3, 3, 3), b.kind, b.params, b.coef, path="extrusion")
    with pytest.raises(hx.SimplificationNotApplicableError):  # anisotropic: general-kernel route
        gram_batched("H1", (2, 3, 2), b.kind, b.params, b.coef, path="extrusion")
    x = extrusion_batch(2, 6)
    x.params[1, 2:10] = x.params[1, [4, 5, 2, 3, 6, 7, 8, 9]]  # swap v00 <-> v10: det < 0
    with pytest.raises(hx.DegenerateMapError):
        gram_batched("H1", (3, 3, 3), x.kind, x.params, x.coef, path="extrusion")


def test_extrusion_host_entry_matches_device_entry():
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.engine import get_engine
    from paper_1711_00984_b200.inputs import dim, extrusion_batch

    b = extrusion_batch(37, 710, variable_coef=True)
    dev, _ = gram_batched("Hcurl", (4, 4, 4), b.kind, b.params, b.coef, path="extrusion")
    N = dim("Hcurl", (4, 4, 4))
    out = np.empty((37, N * (N + 1) // 2))
    get_engine().integrate_host("Hcurl", "extrusion", (4, 4, 4), 5, b.kind, b.params, b.coef, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out, dev.cpu().numpy())


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("orders,L", [((2, 1, 1), 2), ((3, 2, 1), 2), ((4, 2, 3), 3), ((1, 3, 2), 1)])
def test_extrusion_anisotropic_short_rule(space, orders, L, orc):
    """Regression (found by tests/test_gpu_property.py): anisotropic orders with a rule
    shorter than p1 + 1 on the extrusion path -- xi1 must still be integrated exactly
    (simp_*_ext uses F tables in xi1), only (xi2, xi3) use the L-point rule."""
    from paper_1711_00984_b200.inputs import extrusion_batch

    b = extrusion_batch(4, 900 + L + sum(orders), variable_coef=True)
    check_batch(space, "extrusion", orders, L, b, orc)


def test_two_streams_do_not_share_workspace():
    """Calls on distinct streams get distinct scratch buffers (engine.workspace is
    keyed by stream): two general-path batches issued back to back on two streams
    equal the same batches run alone."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b1, b2 = trilinear_batch(64, 71, variable_coef=True), trilinear_batch(64, 72, variable_coef=True)
    ref1, _ = gram_batched("Hdiv", (5, 5, 5), b1.kind, b1.params, b1.coef)
    ref2, _ = gram_batched("H1", (6, 6, 6), b2.kind, b2.params, b2.coef)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        g1, _ = gram_batched("Hdiv", (5, 5, 5), b1.kind, b1.params, b1.coef, stream=s1)
    with torch.cuda.stream(s2):
        g2, _ = gram_batched("H1", (6, 6, 6), b2.kind, b2.params, b2.coef, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(g1, ref1) and torch.equal(g2, ref2)
