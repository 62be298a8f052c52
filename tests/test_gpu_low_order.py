"""The low-order slab kernel (hxg_general_lo.cuh: isotropic p <= hxg_fused_order_max(),
default rule, geometry evaluated in the kernel) through the C ABI against the CPU oracle:
every space and order, batch sizes that do not fill the element slots of a CTA pass
(1, 3, 17, 67 elements), per-node mass weights, the degenerate-map flag of one element
inside a multi-element pass, and agreement with the warp-unit route (HXG_LO=0).

Tolerance: relative Frobenius error per element <= 1e-12 (north_star)."""

import numpy as np
import pytest

from test_gpu_parity import TOL, check_batch, rel_fro

pytestmark = pytest.mark.gpu

SPACES = ("H1", "Hcurl", "Hdiv", "L2")


def test_fused_order_max_is_exported():
    from paper_1711_00984_b200 import _native

    assert _native.lib().hxg_fused_order_max() == 4


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("E", [1, 3, 17])
def test_slab_kernel_ragged_batches(space, p, E, orc):
    """E is not a multiple of the elements per CTA pass: dead slots must neither
    write nor block the pass."""
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(E, 4000 + 10 * p + E, variable_coef=True)
    check_batch(space, "general", (p, p, p), p + 1, b, orc)


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [2, 3, 4])
def test_slab_kernel_matches_warp_unit_route(space, p, monkeypatch):
    """67 elements (several CTA passes, a partial last one) by the slab kernel and by
    the round-1 route (fused v3 at p <= 3, metric pass + v3 at p = 4)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(67, 4100 + p, variable_coef=True)
    a, sa = gram_batched(space, (p, p, p), b.kind, b.params, b.coef)
    monkeypatch.setenv("HXG_LO", "0")
    o, so = gram_batched(space, (p, p, p), b.kind, b.params, b.coef)
    monkeypatch.delenv("HXG_LO")
    torch.cuda.synchronize()
    rel = torch.linalg.norm(a - o, dim=1) / torch.linalg.norm(o, dim=1)
    assert float(rel.max()) <= TOL, (space, p, float(rel.max()))
    assert int(sa.abs().sum()) == 0 and int(so.abs().sum()) == 0


@pytest.mark.parametrize("space", SPACES)
@pytest.mark.parametrize("p", [2, 4])
def test_slab_kernel_per_node_weights(space, p, orc):
    """wgrid (callable mass weights sampled at the tensor nodes, gram.py:78-90)."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim, trilinear_batch

    E, L = 9, p + 1
    b = trilinear_batch(E, 4200 + p)
    wgrid = np.random.default_rng(4200 + p).uniform(0.5, 2.0, (E, L ** 3))
    packed, status = gram_batched(space, (p, p, p), b.kind, b.params, None, rule_order=L, wgrid=wgrid)
    torch.cuda.synchronize()
    got = packed.cpu().numpy()
    ref = orc.gram_batched(space, "general", (p, p, p), L, b.kind, b.params, None, wgrid)
    N = dim(space, (p, p, p))
    worst = max(rel_fro(got[e], ref[e], N, orc) for e in range(E))
    assert worst <= TOL, (space, p, worst)
    assert int(status.abs().sum()) == 0


def test_slab_kernel_flags_the_degenerate_element_only():
    """One inverted element among others in the same CTA pass: its status word carries
    bit 0, its neighbours' stay 0 and their matrices are unaffected."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(11, 4300, variable_coef=True)
    good, s0 = gram_batched("Hdiv", (2, 2, 2), b.kind, b.params, b.coef)
    par = b.params.copy().reshape(11, 8, 3)
    par[5, :, 0] = 1.0 - par[5, :, 0]  # mirror x: det < 0 everywhere
    bad, s1 = gram_batched("Hdiv", (2, 2, 2), b.kind, par.reshape(11, 24), b.coef, check_status=False)
    torch.cuda.synchronize()
    st = s1.cpu().numpy()
    assert int(s0.abs().sum()) == 0
    assert st[5] & 1 and not st[np.arange(11) != 5].any()
    keep = torch.tensor([e for e in range(11) if e != 5], device=good.device)
    assert torch.equal(good[keep], bad[keep])
