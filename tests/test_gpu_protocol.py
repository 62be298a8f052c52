"""Parity protocol of BASELINE.md section 3.5 on the sm_100a path (through the
C ABI), and direct checks of the device 1D tables against the reference's
arrays.

* all 64 elements of config 1; >= 32 elements of every other BASELINE config
  (first, last and seeded picks of the full-size batch);
* >= 8 elements per config-5 sweep order p >= 8, for H1 / H(curl) / H(div) on
  the general and affine paths;
* device Gauss rules, chi / chi' / nu tables and F tables read back from
  hxg_make_tables against tests/golden/golden_ref.npz (quadrature.py:47-66,
  poly1d.py:77-137, 251-266).

Tolerance: relative Frobenius error per element <= 1e-12 (BASELINE.json
north_star); tables <= 2e-16 absolute."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12


def rel_fro(got_packed, ref_packed, N, orc):
    G = orc.unpack(got_packed, N)
    R = orc.unpack(ref_packed, N)
    return np.linalg.norm(G - R) / np.linalg.norm(R)


def protocol_sample(E: int, k: int, seed: int):
    """First, last and seeded picks: k distinct element indices of a batch of E."""
    if E <= k:
        return list(range(E))
    rng = np.random.default_rng(seed)
    pick = {0, E - 1}
    while len(pick) < k:
        pick.add(int(rng.integers(0, E)))
    return sorted(pick)


def _check(wl, b, packed, sample, orc):
    from paper_1711_00984_b200.inputs import dim

    N = dim(wl.space, wl.orders)
    ref = orc.gram_batched(wl.space, wl.path, wl.orders, wl.L, b.kind[sample], b.params[sample],
                           b.coef[sample])
    got = packed[sample].cpu().numpy()
    worst = max(rel_fro(got[i], ref[i], N, orc) for i in range(len(sample)))
    assert worst <= TOL, (wl.name, worst)
    return worst


@pytest.mark.parametrize("name", ["c1_h1_p3_affine", "c2_h1_p5_general", "c3_hcurl_p6_general",
                                  "c3_hcurl_p6_affine", "c4_hdiv_p7_general", "c4_l2_p7_general"])
def test_config_parity_protocol(name, orc):
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import WORKLOADS

    wl = WORKLOADS[name]
    b = wl.batch()
    packed, status = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef, path=wl.path,
                                  rule_order=wl.L)
    torch.cuda.synchronize()
    assert int(status.abs().sum()) == 0
    k = 64 if name == "c1_h1_p3_affine" else 32
    sample = protocol_sample(b.size, k, seed=sum(name.encode()))
    assert len(sample) == min(k, b.size)
    _check(wl, b, packed, sample, orc)


@pytest.mark.parametrize("space", ["H1", "Hcurl", "Hdiv"])
@pytest.mark.parametrize("path", ["general", "affine"])
@pytest.mark.parametrize("p", [8, 9, 10])
def test_sweep_high_order_parity(space, path, p, orc):
    """Config-5 sweep orders p >= 8: the seeded sweep generator (seed 4), a
    multi-wave batch, >= 8 elements checked (first, last, seeded picks)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import SWEEP_WORKLOADS

    wl = SWEEP_WORKLOADS[f"c5_{space.lower()}_p{p}_{path}"]
    E = min(wl.E, 1200)
    b = wl.batch(E)
    packed, status = gram_batched(wl.space, wl.orders, b.kind, b.params, b.coef, path=wl.path,
                                  rule_order=wl.L)
    torch.cuda.synchronize()
    assert int(status.abs().sum()) == 0
    _check(wl, b, packed, protocol_sample(E, 8, seed=p), orc)


def _tables(L, nodes=None, weights=None):
    import torch

    from paper_1711_00984_b200.engine import get_engine

    t = get_engine().tables(L, nodes, weights)
    torch.cuda.synchronize()
    return t.cpu().numpy()


def test_device_gauss_rules_match_reference(golden):
    """hxg_make_tables(L) nodes / weights vs the reference's gauss_rule(L), L = 1..16."""
    from paper_1711_00984_b200 import _native as nat

    worst = 0.0
    for L in range(1, 17):
        t = _tables(L)
        n = t[nat.TAB_NODES:nat.TAB_NODES + L]
        w = t[nat.TAB_WTS:nat.TAB_WTS + L]
        worst = max(worst, np.abs(n - golden[f"rule_{L}_nodes"]).max(),
                    np.abs(w - golden[f"rule_{L}_weights"]).max())
        assert np.all(t[nat.TAB_NODES + L:nat.TAB_NODES + nat.LT] == 0.0)
    assert worst <= 2e-16, worst


def test_device_shape_tables_match_reference(golden):
    """chi_k / chi'_k / nu_k (k <= 12) evaluated on the device at the golden points
    (user-rule path of hxg_make_tables) vs poly1d.shape1_h1 / shape1_l2."""
    from paper_1711_00984_b200 import _native as nat

    pts = golden["shape_pts"]
    L = pts.size
    t = _tables(L, pts, np.full(L, 1.0 / L))
    T = t[nat.TAB_T:nat.TAB_T + 2 * nat.KT * nat.LT].reshape(2, nat.KT, nat.LT)
    chi = T[0, :13, :L].T
    dchi = T[1, :13, :L].T
    assert np.abs(chi - golden["shape_chi"]).max() <= 2e-16
    assert np.abs(dchi - golden["shape_dchi"]).max() <= 2e-16
    # nu_i = P_i = chi'_{i+1} (poly1d.py:125-137, the tables' shift)
    assert np.abs(T[1, 1:13, :L].T - golden["shape_nu"]).max() <= 2e-16
    np.testing.assert_array_equal(t[nat.TAB_NODES:nat.TAB_NODES + L], pts)


def test_device_ftables_match_reference(golden):
    """Closed-form F tables (poly1d.py:140-266) vs ftable(12).stacked."""
    from paper_1711_00984_b200 import _native as nat

    t = _tables(4)
    F = t[nat.TAB_F:nat.TAB_F + 4 * nat.KT * nat.KT].reshape(4, nat.KT, nat.KT)
    assert np.abs(F[:, :13, :13] - golden["ftable_12"]).max() <= 2e-16


# ---------------------------------------------------------------------------
# drop-in entry points not covered elsewhere (gram.py:101-124, 235-253)
# ---------------------------------------------------------------------------
def test_gram_block_replication():
    """test_gram.py:215-229 pattern: block-diagonal copies, off-diagonal exactly zero."""
    import paper_1711_00984_b200 as hx

    sig = hx.SpaceSignature("H1", (1, 1, 1))
    emap = hx.identity_map()
    base = hx.gram(sig, emap, "conventional")
    b3 = hx.gram_block(sig, emap, "conventional", copies=3)
    assert b3.matrix.shape == (24, 24)
    np.testing.assert_array_equal(b3.matrix[:8, :8], base.matrix)
    np.testing.assert_array_equal(b3.matrix[8:16, 8:16], base.matrix)
    np.testing.assert_array_equal(b3.matrix[16:, 16:], base.matrix)
    assert np.all(b3.matrix[:8, 8:] == 0.0) and np.all(b3.matrix[8:, :8] == 0.0)
    b1 = hx.gram_block(sig, emap, "conventional", copies=1)
    np.testing.assert_array_equal(b1.matrix, base.matrix)
    sig_v = hx.SpaceSignature("Hdiv", (1, 1, 1))
    assert hx.gram_block(sig_v, emap, copies=3).matrix.shape == (18, 18)
    bt = hx.gram_block(hx.SpaceSignature("Hcurl", (2, 2, 2)), hx.preset_map("trilinear"),
                       "tensorized", copies=3, rule_order=3)
    assert bt.counters == hx.gram(hx.SpaceSignature("Hcurl", (2, 2, 2)), hx.preset_map("trilinear"),
                                  "tensorized", rule_order=3).counters
    with pytest.raises(ValueError):
        hx.gram_block(sig, emap, copies=2)


def test_gram_conventional_matches_golden_and_tensorized(golden, orc):
    """gram_conventional through the drop-in: the same tensor-rule integral as
    gram_tensorized (test_gram.py:91-101), a user Rule3D used as given, the
    conventional counters, and a non-tensor Rule3D rejected."""
    import paper_1711_00984_b200 as hx

    em = hx.preset_map("trilinear")
    for space in ("H1", "Hcurl", "Hdiv", "L2"):
        for orders in ((1, 2, 3), (3, 3, 3)):
            sig = hx.SpaceSignature(space, orders)
            L = hx.default_rule_order(space, orders)
            conv = hx.gram_conventional(sig, em, hx.tensor_rule(L))
            tens = hx.gram_tensorized(sig, em, hx.gauss_rule(L))
            np.testing.assert_array_equal(conv.matrix, tens.matrix)
            N = conv.matrix.shape[0]
            assert conv.counters == hx.OpCounters(L ** 3 * N * (N + 1) // 2, L ** 3, 0, L ** 3)
    # a non-Gauss tensor rule is integrated with its own nodes and weights
    n = np.array([0.15, 0.5, 0.85, 0.95])
    w = np.array([0.3, 0.3, 0.25, 0.15])
    pts = np.stack(np.meshgrid(n, n, n, indexing="ij"), axis=-1).reshape(-1, 3)
    wts = np.einsum("i,j,k->ijk", w, w, w).reshape(-1)
    sig = hx.SpaceSignature("Hdiv", (2, 2, 2))
    got = hx.gram_conventional(sig, em, hx.Rule3D(pts, wts, 4)).matrix
    ref, _ = orc.gram_full("Hdiv", "general", (2, 2, 2), 4, em.kind_code, em.params, 1.0,
                           nodes=n, weights=w)
    assert np.linalg.norm(got - ref) <= TOL * np.linalg.norm(ref)
    bad = pts.copy()
    bad[5, 0] = 0.33
    with pytest.raises(ValueError):
        hx.gram_conventional(sig, em, hx.Rule3D(bad, wts, 4))


# ---------------------------------------------------------------------------
# host-buffer C-ABI entry = the reference's kernel seam (gram.py:154-157)
# ---------------------------------------------------------------------------
def test_host_entry_user_rule_and_weight_grid(golden, orc):
    """hxg_gram_batched_host with the seam's full argument list: a non-Gauss
    Rule1D (nodes, weights) and sampled mass weights (wgrid) -- the golden
    callable-weight cases of the reference, and a user rule vs the oracle."""
    from conftest import golden_cases
    from paper_1711_00984_b200.engine import get_engine
    from paper_1711_00984_b200.inputs import packed_size, trilinear_batch

    eng = get_engine()
    n = 0
    for c in golden_cases(golden):
        if c["wgrid"] is None or c["path"] != "general":
            continue
        L = c["L"]
        out = np.empty((1, packed_size(c["space"], c["orders"])))
        eng.integrate_host(c["space"], "general", c["orders"], L, np.array([c["kind"]]),
                           c["params"].reshape(1, 24), None, out, wgrid=c["wgrid"].reshape(1, -1))
        ref = c["packed"]
        assert np.linalg.norm(out[0] - ref) <= TOL * np.linalg.norm(ref), (c["space"], c["orders"])
        n += 1
    assert n >= 4
    # a user rule (non-Gauss nodes and weights) plus a per-element weight grid
    nodes = np.array([0.04, 0.2, 0.45, 0.6, 0.8, 0.97])
    wts = np.array([0.1, 0.2, 0.2, 0.2, 0.2, 0.1])
    b = trilinear_batch(6, 77, variable_coef=True)
    rng = np.random.default_rng(5)
    wgrid = rng.uniform(0.5, 2.0, (6, 6 ** 3))
    for space, orders in (("H1", (3, 3, 3)), ("Hcurl", (2, 3, 4)), ("Hdiv", (5, 5, 5))):
        out = np.empty((6, packed_size(space, orders)))
        st = np.zeros(6, np.int32)
        eng.integrate_host(space, "general", orders, 6, b.kind, b.params, b.coef, out, st,
                           nodes=nodes, weights=wts, wgrid=wgrid)
        assert st.sum() == 0
        for e in range(6):
            R, _ = orc.gram_full(space, "general", orders, 6, b.kind[e], b.params[e], 1.0,
                                 wgrid=wgrid[e], nodes=nodes, weights=wts)
            G = orc.unpack(out[e], R.shape[0])
            assert np.linalg.norm(G - R) <= TOL * np.linalg.norm(R), (space, e)


def test_host_entry_raises_without_status_array():
    """A flagged element is an error even when the caller passes no status array
    (the reference raises before returning a matrix)."""
    import paper_1711_00984_b200 as hx
    from paper_1711_00984_b200.engine import get_engine
    from paper_1711_00984_b200.inputs import packed_size, trilinear_batch

    eng = get_engine()
    b = trilinear_batch(3, 9)
    par = b.params.copy().reshape(3, 8, 3)
    par[1, :, 0] = 1.0 - par[1, :, 0]  # element 1 mirrored: det < 0
    out = np.empty((3, packed_size("H1", (3, 3, 3))))
    with pytest.raises(hx.DegenerateMapError):
        eng.integrate_host("H1", "general", (3, 3, 3), 4, b.kind, par.reshape(3, 24), None, out)
    st = np.zeros(3, np.int32)
    with pytest.raises(hx.DegenerateMapError) as ei:
        eng.integrate_host("H1", "general", (3, 3, 3), 4, b.kind, par.reshape(3, 24), None, out, st)
    assert list(np.nonzero(st)[0]) == [1] and ei.value.point == (1,)
    with pytest.raises(hx.SimplificationNotApplicableError):
        eng.integrate_host("H1", "affine", (3, 3, 3), 1, b.kind, b.params, None, out)
    with pytest.raises(ValueError):  # sampled weights on a simplified path (gram.py:93-98)
        eng.integrate_host("H1", "extrusion", (3, 3, 3), 4, b.kind, b.params, None, out,
                           wgrid=np.ones((3, 64)))


def test_stream_argument_without_current_stream_context():
    """integrate(stream=s) while s is NOT the current stream: inputs produced on
    the current stream are waited for, the status is read on s."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(64, 31, variable_coef=True)
    ref, _ = gram_batched("Hcurl", (5, 5, 5), b.kind, b.params, b.coef)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    for _ in range(3):
        kind = torch.as_tensor(b.kind).cuda()
        params = torch.as_tensor(b.params).cuda() * 1.0  # produced on the current stream
        coef = torch.full((64,), 0.0, dtype=torch.float64, device="cuda") + torch.as_tensor(b.coef).cuda()
        got, st = gram_batched("Hcurl", (5, 5, 5), kind, params, coef, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        assert torch.equal(got, ref)
        assert int(st.abs().sum()) == 0
    # deferred status: no host sync inside, raised later on request
    from paper_1711_00984_b200.engine import get_engine

    par = b.params.copy().reshape(64, 8, 3)
    par[7, :, 0] = 1.0 - par[7, :, 0]
    _, st = gram_batched("H1", (4, 4, 4), b.kind, par.reshape(64, 24), b.coef, check_status=False)
    import paper_1711_00984_b200 as hx

    with pytest.raises(hx.DegenerateMapError):
        get_engine().raise_for_status(st, "general")
