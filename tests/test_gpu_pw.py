"""Round-2 kernels on the GPU, through the C ABI, against the CPU oracle:

* the warp-owned P-form general-map kernel (hxg_general_pw.cuh) -- the default
  route at p >= 8 (H1, H(curl), H(div)), forced at every order it supports with
  HXG_PW=1 -- including small / ragged batches (fewer work items than CTAs) and
  its K-digit and 8-digit-group shapes;
* the specialized metric kernel (hxg_metric.cuh): fields equal to the generic
  metric kernel's, status words written whole (no memset before it), degenerate
  maps flagged.

Tolerance: relative Frobenius error per element <= 1e-12 (north_star)."""

import ctypes

import numpy as np
import pytest

from test_gpu_parity import TOL, check_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("space", ["H1", "Hcurl", "Hdiv", "L2"])
@pytest.mark.parametrize("p", [4, 5, 6, 7, 8, 9, 10])
def test_pw_kernel_every_order(space, p, monkeypatch, orc):
    from paper_1711_00984_b200.inputs import trilinear_batch

    monkeypatch.setenv("HXG_PW", "1")
    b = trilinear_batch(2, 900 + p, variable_coef=True)
    check_batch(space, "general", (p, p, p), p + 1, b, orc)


@pytest.mark.parametrize("space,p", [("Hdiv", 8), ("Hcurl", 9), ("H1", 10)])
@pytest.mark.parametrize("E", [1, 3, 7])
def test_pw_small_batches(space, p, E, orc):
    """Fewer (element, unit) items than CTAs x warps: the per-CTA item ranges
    [c T / G, (c + 1) T / G) must still cover every unit exactly once."""
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(E, 950 + E, variable_coef=True)
    check_batch(space, "general", (p, p, p), p + 1, b, orc)


def test_pw_matches_v2_on_a_larger_batch(monkeypatch):
    """PW (default at p = 8) and the CTA-chunked v2 kernel agree on 64 elements."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(64, 77, variable_coef=True)
    for space in ("H1", "Hcurl", "Hdiv"):
        a, _ = gram_batched(space, (8, 8, 8), b.kind, b.params, b.coef)
        monkeypatch.setenv("HXG_PW", "0")
        v2, _ = gram_batched(space, (8, 8, 8), b.kind, b.params, b.coef)
        monkeypatch.delenv("HXG_PW")
        torch.cuda.synchronize()
        rel = torch.linalg.norm(a - v2, dim=1) / torch.linalg.norm(v2, dim=1)
        assert float(rel.max()) <= TOL, space


def _metric(space, p, L, b, status_fill, monkeypatch=None, generic=False):
    import torch

    from paper_1711_00984_b200 import _native
    from paper_1711_00984_b200.engine import get_engine

    if generic:
        monkeypatch.setenv("HXG_FORCE_GENERIC", "1")
    eng = get_engine()
    lib = _native.lib()
    dev = eng.device
    sc = _native.SPACE_CODES[space]
    kind = torch.as_tensor(b.kind, dtype=torch.int32).to(dev)
    params = torch.as_tensor(b.params).to(dev)
    coef = torch.as_tensor(b.coef).to(dev)
    per = lib.hxg_workspace_size(sc, 0, p, p, p, L, 1)
    met = torch.empty(b.size * per // 8, dtype=torch.float64, device=dev)
    status = torch.full((b.size,), status_fill, dtype=torch.int32, device=dev)
    tab = eng.tables(L)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    rc = lib.hxg_metric_batched(sc, p, p, p, L, b.size, vp(kind), vp(params), vp(coef), None, vp(tab),
                                vp(met), vp(status), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    if generic:
        monkeypatch.delenv("HXG_FORCE_GENERIC")
    return met.cpu().numpy(), status.cpu().numpy()


@pytest.mark.parametrize("space", ["H1", "Hcurl", "Hdiv", "L2"])
def test_specialized_metric_equals_generic(space, monkeypatch):
    from paper_1711_00984_b200.inputs import affine_batch, trilinear_batch

    tb = trilinear_batch(9, 31, variable_coef=True)
    ab = affine_batch(4, 32, variable_coef=True)
    for b in (tb, ab):
        for p in (4, 7, 10):
            m1, s1 = _metric(space, p, p + 1, b, 0x7F7F)
            m0, s0 = _metric(space, p, p + 1, b, 0, monkeypatch, generic=True)
            np.testing.assert_allclose(m1, m0, rtol=1e-13, atol=1e-15 * np.abs(m0).max())
            # the specialized kernel writes every status word (the prefill is gone)
            assert (s1 == 0).all() and (s0 == 0).all()


def test_specialized_metric_flags_degenerate_element():
    from paper_1711_00984_b200.inputs import trilinear_batch

    b = trilinear_batch(5, 41)
    b.params[3] = b.params[3].reshape(8, 3)[[1, 0, 3, 2, 5, 4, 7, 6]].reshape(24)  # mirror: det < 0
    _, s = _metric("Hdiv", 6, 7, b, 0x55)
    assert s.tolist() == [0, 0, 0, 1, 0]
