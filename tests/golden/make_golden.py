"""Generate the golden vectors that pin the CPU oracle (and the CUDA path)
to the reference implementation.

Run in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every array is produced by the reference's own public API
(/root/reference/pkg/src/hexgram: quadrature.gauss_rule, poly1d.shape1_h1 /
shape1_l2 / ftable, _kernels._geom_full, gram.gram_tensorized /
gram_simplified / _weight_grid).  The GPU box has no /root/reference, so the
tests read only the .npz written here.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import hexgram as hg  # noqa: E402
from hexgram import _kernels as K  # noqa: E402
from hexgram.geometry import preset_map  # noqa: E402
from hexgram.gram import _weight_grid  # noqa: E402

from paper_1711_00984_b200.inputs import WORKLOADS, dim  # noqa: E402

OUT = os.path.join(HERE, "golden_ref.npz")
SPACES = ("H1", "Hcurl", "Hdiv", "L2")
MAPS = ("identity", "diagonal-affine", "general-affine", "trilinear")
PATHS = ("general", "affine", "extrusion")  # meta[1]


def packed(G):
    return G[np.triu_indices(G.shape[0])]


def main():
    d = {}
    # 1D rules, quadrature.py:47-66
    for L in range(1, 17):
        r = hg.gauss_rule(L)
        d[f"rule_{L}_nodes"] = r.nodes
        d[f"rule_{L}_weights"] = r.weights
    # 1D shape tables, poly1d.py:77-99
    pts = np.array([0.0, 0.05, 0.21132486540518713, 0.5, 0.77, 0.93, 1.0])
    d["shape_pts"] = pts
    d["shape_chi"] = np.array([hg.shape1_h1(12, x).chi for x in pts])
    d["shape_dchi"] = np.array([hg.shape1_h1(12, x).dchi for x in pts])
    d["shape_nu"] = np.array([hg.shape1_l2(12, x) for x in pts])
    # F tables, poly1d.py:251-266
    d["ftable_12"] = hg.ftable(12).stacked
    # geometry, _kernels.py:100-118 (params of the presets + seeded maps)
    gk, gp, gx, gJ, gJi, gdet = [], [], [], [], [], []
    rng = np.random.default_rng(123)
    emaps = [preset_map(m) for m in MAPS + ("extrusion",)]
    emaps += [hg.trilinear_map(WORKLOADS["c3_hcurl_p6_general"].batch(3).params[i]) for i in range(3)]
    for em in emaps:
        for _ in range(3):
            xi = rng.uniform(0, 1, 3)
            J = np.empty((3, 3))
            Ji = np.empty((3, 3))
            det = K._geom_full(em.kind_code, em.params, xi[0], xi[1], xi[2], J, Ji)
            gk.append(em.kind_code)
            gp.append(em.params)
            gx.append(xi)
            gJ.append(J)
            gJi.append(Ji)
            gdet.append(det)
    d.update(geo_kind=np.array(gk, np.int32), geo_params=np.array(gp), geo_xi=np.array(gx),
             geo_J=np.array(gJ), geo_Jinv=np.array(gJi), geo_det=np.array(gdet))

    # Gram matrices through the reference's public entry points
    cases = []
    for space in SPACES:
        for orders in [(1, 1, 1), (2, 2, 2), (2, 3, 2), (1, 2, 3), (3, 2, 3), (3, 3, 3), (2, 3, 4)]:
            for mname in MAPS:
                em = preset_map(mname)
                sig = hg.SpaceSignature(space, orders)
                L = max(orders) + 1
                coef = 1.0 if orders[0] != 2 else 1.7
                res = hg.gram_tensorized(sig, em, hg.gauss_rule(L), "alternative",
                                         mass_weight=coef)
                cases.append((space, "general", orders, L, em.kind_code, em.params, coef, None,
                              res.matrix, res.counters.accumulations))
                if hg.classify(em) == "constant-jacobian":
                    res = hg.gram_simplified(sig, em, mass_weight=coef)
                    cases.append((space, "affine", orders, L, em.kind_code, em.params, coef,
                                  None, res.matrix, res.counters.accumulations))
    # simplified extrusion path (gram.py:192-203 -> simp_*_ext, _kernels.py:1405-1764):
    # the preset map and a seeded random extrusion, default rule (L2: L = max p)
    rng_x = np.random.default_rng(11)
    quad = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    ext_maps = [preset_map("extrusion"),
                hg.extrusion_map(0.8, 0.3, quad + rng_x.uniform(-0.15, 0.15, (4, 2)))]
    for space in SPACES:
        for orders in [(1, 1, 1), (2, 2, 2), (2, 3, 2), (1, 2, 3), (3, 2, 3), (3, 3, 3), (2, 3, 4)]:
            for k, em in enumerate(ext_maps):
                sig = hg.SpaceSignature(space, orders)
                coef = 1.0 if k == 0 else 1.4
                L = hg.default_rule_order(space, orders)
                res = hg.gram_simplified(sig, em, mass_weight=coef)
                cases.append((space, "extrusion", orders, L, em.kind_code, em.params, coef, None,
                              res.matrix, res.counters.accumulations))
    # reference default rule order for L2 is max(p) (quadrature.py:86-89)
    for orders in [(2, 2, 2), (3, 2, 3)]:
        em = preset_map("trilinear")
        sig = hg.SpaceSignature("L2", orders)
        res = hg.gram_tensorized(sig, em)
        cases.append(("L2", "general", orders, max(orders), em.kind_code, em.params, 1.0, None,
                      res.matrix, res.counters.accumulations))
    # variable mass weight sampled by the reference (gram.py:78-90; test_gram.py:240-253)
    for space in SPACES:
        em = preset_map("trilinear")
        sig = hg.SpaceSignature(space, (2, 2, 2))
        L = 4
        w = lambda x: 1.0 + x[0] ** 2 + 0.5 * x[1]  # noqa: E731
        rule = hg.gauss_rule(L)
        res = hg.gram_tensorized(sig, em, rule, "alternative", mass_weight=w)
        wg = _weight_grid(em, rule.nodes, w)
        cases.append((space, "general", (2, 2, 2), L, em.kind_code, em.params, 1.0, wg,
                      res.matrix, res.counters.accumulations))
    for i, (space, path, orders, L, kind, par, coef, wg, G, acc) in enumerate(cases):
        pre = f"case{i:03d}"
        d[pre + "_meta"] = np.array([SPACES.index(space), PATHS.index(path), *orders, L, kind, acc],
                                    np.int64)
        d[pre + "_params"] = par
        d[pre + "_coef"] = np.array([coef])
        if wg is not None:
            d[pre + "_wgrid"] = wg.reshape(-1)
        d[pre + "_packed"] = packed(G)
    d["n_cases"] = np.array([len(cases)])

    # BASELINE.json config samples: the seeded batches, reference kernels called
    # the way BASELINE.md section 3 prescribes.
    rng = np.random.default_rng(7)
    for name, wl in WORKLOADS.items():
        nel = 8 if name == "c1_h1_p3_affine" else 1
        b = wl.batch(max(nel, 4))
        N = dim(wl.space, wl.orders)
        for e in range(nel):
            em = hg.ElementMap("trilinear" if b.kind[e] == 4 else "general-affine", b.params[e])
            sig = hg.SpaceSignature(wl.space, wl.orders)
            if wl.path == "general":
                G = hg.gram_tensorized(sig, em, hg.gauss_rule(wl.L), "alternative",
                                       mass_weight=float(b.coef[e])).matrix
            else:
                G = hg.gram_simplified(sig, em, mass_weight=float(b.coef[e])).matrix
            pk = packed(G)
            pre = f"{name}_e{e}"
            if N <= 64:
                d[pre + "_packed"] = pk
            else:
                idx = np.sort(rng.choice(pk.size, 4096, replace=False))
                idx = np.unique(np.concatenate([idx, [0, pk.size - 1]]))
                d[pre + "_idx"] = idx
                d[pre + "_val"] = pk[idx]
            d[pre + "_fro"] = np.array([np.linalg.norm(G)])
            d[pre + "_sum"] = np.array([pk.sum()])
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(cases), "cases")


if __name__ == "__main__":
    main()
