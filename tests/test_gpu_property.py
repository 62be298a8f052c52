"""Randomised parity (hypothesis): arbitrary small (space, orders, path, rule,
map kind, coefficient) draws through the C ABI against the CPU oracle, plus
mixed-kind batches.  Complements the fixed grids of test_gpu_parity.py with
combinations nobody listed by hand (anisotropic orders on every path, rules
with L != p + 1, kinds 0-4 in one batch).  Tolerance: relative Frobenius error
per element <= 1e-12 (BASELINE north_star)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

TOL = 1e-12
SPACES = ("H1", "Hcurl", "Hdiv", "L2")
CUBE = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], float)


def _params(kind: int, rng) -> np.ndarray:
    """Element-map parameters of geometry.py:83-119 for `kind`, det J > 0."""
    p = np.zeros(24)
    if kind == 1:
        p[0:3] = rng.uniform(0.5, 2.0, 3)
    elif kind == 2:
        p[0:9] = (np.eye(3) + rng.uniform(-0.2, 0.2, (3, 3))).reshape(9)
        p[9:12] = rng.uniform(0, 1, 3)
    elif kind == 3:  # extrusion: x1 scale + a perturbed unit square in (x2, x3)
        p[0] = rng.uniform(0.5, 2.0)
        sq = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
        p[2:10] = (sq + rng.uniform(-0.1, 0.1, (4, 2))).reshape(8)
    elif kind == 4:
        p[:] = (CUBE + rng.uniform(-0.1, 0.1, (8, 3))).reshape(24)
    return p


@settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))
@given(space=st.sampled_from(SPACES),
       orders=st.tuples(st.integers(1, 5), st.integers(1, 5), st.integers(1, 5)),
       path=st.sampled_from(["general", "affine", "extrusion"]),
       dL=st.integers(-1, 2), E=st.integers(1, 5), seed=st.integers(0, 2 ** 31 - 1),
       mixed=st.booleans())
def test_random_cases_vs_oracle(space, orders, path, dL, E, seed, mixed, orc):
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim

    rng = np.random.default_rng(seed)
    max_kind = {"general": 4, "affine": 2, "extrusion": 3}[path]
    kinds = rng.integers(0, max_kind + 1, E) if mixed else np.full(E, max_kind)
    kind = kinds.astype(np.int32)
    params = np.stack([_params(int(k), rng) for k in kind])
    coef = rng.uniform(0.5, 2.0, E)
    L = max(1, max(orders) + 1 + dL)
    packed, status = gram_batched(space, orders, kind, params, coef, path=path,
                                  rule_order=L if path != "affine" else None)
    torch.cuda.synchronize()
    assert int(status.abs().sum()) == 0
    got = packed.cpu().numpy()
    ref = orc.gram_batched(space, path, orders, L if path != "affine" else 1, kind, params, coef)
    N = dim(space, orders)
    for e in range(E):
        G, R = orc.unpack(got[e], N), orc.unpack(ref[e], N)
        rel = np.linalg.norm(G - R) / np.linalg.norm(R)
        assert rel <= TOL, (space, orders, path, L, int(kind[e]), rel)


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(space=st.sampled_from(SPACES),
       orders=st.tuples(st.integers(1, 4), st.integers(1, 4), st.integers(1, 4)),
       dL=st.integers(0, 2), E=st.integers(1, 4), seed=st.integers(0, 2 ** 31 - 1))
def test_random_wgrid_vs_oracle(space, orders, dL, E, seed, orc):
    """Per-node mass weights (gram.py:78-90, host-sampled callables) on the general path."""
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim

    rng = np.random.default_rng(seed)
    kind = np.full(E, 4, np.int32)
    params = np.stack([_params(4, rng) for _ in range(E)])
    L = max(orders) + 1 + dL
    wgrid = rng.uniform(0.5, 2.0, (E, L ** 3))
    packed, status = gram_batched(space, orders, kind, params, None, path="general",
                                  rule_order=L, wgrid=wgrid)
    torch.cuda.synchronize()
    got = packed.cpu().numpy()
    ref = orc.gram_batched(space, "general", orders, L, kind, params, None, wgrid)
    N = dim(space, orders)
    for e in range(E):
        G, R = orc.unpack(got[e], N), orc.unpack(ref[e], N)
        assert np.linalg.norm(G - R) / np.linalg.norm(R) <= TOL


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(m=st.integers(1, 300), n=st.integers(1, 80), E=st.integers(1, 3),
       seed=st.integers(0, 2 ** 31 - 1), with_l=st.booleans())
def test_random_condense_vs_oracle(m, n, E, seed, with_l, orc):
    """Batched static condensation (dpg.py:348-357) at arbitrary sizes (panel
    remainders, m < 32, m + n + 1 across tile boundaries)."""
    from paper_1711_00984_b200.dpg import condense_batched

    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((E, m, m))
    G = Q @ Q.transpose(0, 2, 1) / m + np.eye(m)[None]
    B = rng.standard_normal((E, m, n))
    l = rng.standard_normal((E, m)) if with_l else None
    iu = np.triu_indices(m)
    A, rhs, st_ = condense_batched(G[:, iu[0], iu[1]], B, l)
    assert int(st_.abs().sum()) == 0
    A, rhs = A.cpu().numpy(), rhs.cpu().numpy()
    for e in range(E):
        Ar, rr = orc.condense(G[e], B[e], l[e] if with_l else np.zeros(m))
        assert np.linalg.norm(A[e] - Ar) <= TOL * np.linalg.norm(Ar)
        if with_l:
            assert np.linalg.norm(rhs[e] - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300)
        else:
            assert not rhs[e].any()


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(p0=st.integers(1, 4), dp=st.integers(1, 3), kind=st.integers(0, 4), E=st.integers(1, 3),
       seed=st.integers(0, 2 ** 31 - 1), pairing=st.sampled_from(["velocity", "pressure"]))
def test_random_acoustics_vs_oracle(p0, dp, kind, E, seed, pairing, orc):
    """Ultraweak-acoustics stiffness and load (dpg.py:234-302) for random orders and
    map kinds (the i3 slabs of the block kernel cover the higher orders)."""
    from paper_1711_00984_b200.dpg import acoustics_batched

    rng = np.random.default_rng(seed)
    pr = p0 + dp
    L = pr + 1
    kinds = np.full(E, kind, np.int32)
    params = np.stack([_params(kind, rng) for _ in range(E)])
    fg = rng.uniform(-1.0, 1.0, (E, L ** 3))
    Bre, Bim, B2, lre, st_ = acoustics_batched(p0, pr, 1.1, kinds, params, fg, pairing=pairing)
    Bre, Bim, B2, lre = (t.cpu().numpy() for t in (Bre, Bim, B2, lre))
    for e in range(E):
        Rre, Rim = orc.acoustics_stiffness(p0, pr, 1.1, kind, params[e])
        R = np.block([[Rre, -Rim], [Rim, Rre]])
        assert np.linalg.norm(B2[e] - R) <= TOL * np.linalg.norm(R)
        rl = orc.acoustics_load(p0, pr, kind, params[e], fg[e], pairing)
        assert np.linalg.norm(lre[e][: rl.size] - rl) <= TOL * max(np.linalg.norm(rl), 1e-300)
