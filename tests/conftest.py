import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden_ref.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    oracle.lib()
    return oracle


def golden_cases(g):
    """Decode the reference Gram cases written by tests/golden/make_golden.py."""
    spaces = ("H1", "Hcurl", "Hdiv", "L2")
    out = []
    for i in range(int(g["n_cases"][0])):
        pre = f"case{i:03d}"
        meta = g[pre + "_meta"]
        out.append(dict(
            space=spaces[int(meta[0])], path=("general", "affine", "extrusion")[int(meta[1])],
            orders=tuple(int(x) for x in meta[2:5]), L=int(meta[5]), kind=int(meta[6]),
            acc=int(meta[7]), params=g[pre + "_params"], coef=float(g[pre + "_coef"][0]),
            wgrid=g[pre + "_wgrid"] if (pre + "_wgrid") in g.files else None,
            packed=g[pre + "_packed"]))
    return out
