"""Golden vectors for the DPG-layer consumers of the Gram kernels
(SURVEY 8(f) rows 2-3): the adjoint-graph Gram (dpg.py:179-231, including the
closed-form cross block dpg.py:155-176) and static condensation
(dpg.py:348-357), produced by the reference itself.

Run in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_dpg.py

Writes tests/golden/golden_dpg.npz (read by tests/test_dpg_*.py on the GPU
box, which has no /root/reference).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import hexgram as hg  # noqa: E402
from hexgram import dpg  # noqa: E402
from hexgram.geometry import preset_map  # noqa: E402

OUT = os.path.join(HERE, "golden_dpg.npz")


def seeded_maps():
    rng = np.random.default_rng(77)
    A = np.eye(3) + rng.uniform(-0.2, 0.2, (3, 3))
    aff = hg.general_affine_map(A, rng.uniform(0, 1, 3))
    verts = np.array([[k & 1, (k >> 1) & 1, (k >> 2) & 1] for k in range(8)], float)
    tri = hg.trilinear_map(verts + rng.uniform(-0.1, 0.1, (8, 3)))
    return {"identity": preset_map("identity"), "affine": aff, "trilinear": tri,
            "extrusion": preset_map("extrusion")}


def main():
    d = {}
    maps = seeded_maps()
    for name, em in maps.items():
        d[f"map_{name}_kind"] = np.array(em.kind_code)
        d[f"map_{name}_params"] = em.params
    # cross block alone (dpg.py:155-176)
    for pr, om in ((1, 1.0), (2, 2.5), (3, 0.7)):
        d[f"mixed_{pr}_{om}"] = dpg._graph_mixed_ftables(pr, om)
    # adjoint-graph Gram, real block form (dpg.py:179-231)
    cases = []
    for pr in (1, 2):
        for name in maps:
            backends = ["tensorized", "conventional"]
            if name != "trilinear":
                backends.append("simplified")
            for be in backends:
                for inc in (True, False):
                    if not inc and be != "tensorized":
                        continue
                    r = dpg.adjoint_graph_gram(pr, 2.0, 0.5, maps[name], be, include_mixed=inc)
                    key = f"graph_{pr}_{name}_{be}_{int(inc)}"
                    d[key] = r.matrix
                    d[key + "_acc"] = np.array(r.counters.accumulations)
                    cases.append(key)
    d["graph_cases"] = np.array(cases)
    # condensation (dpg.py:348-357) of the reference's own element systems
    ccases = []

    def source(x):
        return np.sin(3.0 * x[0]) + x[1] * x[2] + 0.5

    for p0, dp in ((1, 1), (2, 1), (1, 2)):
        for name in ("identity", "trilinear"):
            sys_ = dpg.poisson_primal_element(p0, dp, 1.0, source, maps[name], "tensorized")
            A, rhs = dpg.condense(sys_)
            key = f"poisson_{p0}_{dp}_{name}"
            d[key + "_G"], d[key + "_B"], d[key + "_l"] = sys_.G, sys_.B, sys_.l
            d[key + "_A"], d[key + "_rhs"] = A, rhs
            ccases.append(key)
    prob = dpg.UltraweakAcousticsProblem(omega=2.0, alpha=0.5, f=1.0)
    for p0, dp in ((1, 1),):
        for name in ("identity", "affine"):
            sys_ = dpg.acoustics_ultraweak_element(prob, p0, dp, maps[name], "tensorized")
            A, rhs = dpg.condense(sys_)
            key = f"acoustics_{p0}_{dp}_{name}"
            d[key + "_G"], d[key + "_B"], d[key + "_l"] = sys_.G, sys_.B, sys_.l
            d[key + "_A"], d[key + "_rhs"] = A, rhs
            ccases.append(key)
    d["condense_cases"] = np.array(ccases)
    # ultraweak acoustics stiffness + load (dpg.py:234-336): B (real block form), l
    acases = []
    for pairing in ("velocity", "pressure"):
        prob = dpg.UltraweakAcousticsProblem(omega=1.7, alpha=0.3, f=source, load_pairing=pairing)
        for p0, dp in ((1, 1), (2, 1), (1, 2), (2, 2)):
            for name in ("identity", "affine", "trilinear", "extrusion"):
                if pairing == "pressure" and name != "trilinear":
                    continue
                sys_ = dpg.acoustics_ultraweak_element(prob, p0, dp, maps[name], "tensorized")
                key = f"ac_{pairing}_{p0}_{dp}_{name}"
                d[key + "_B"], d[key + "_l"] = sys_.B, sys_.l
                if p0 == 1 and dp == 1:
                    d[key + "_G"] = sys_.G
                acases.append(key)
    d["acoustics_cases"] = np.array(acases)
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, len(cases), "graph cases,", len(ccases), "condensation cases,",
          len(acases), "acoustics cases")


if __name__ == "__main__":
    main()
