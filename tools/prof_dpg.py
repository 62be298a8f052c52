"""Run each DPG-layer kernel once on a bench-sized batch (for ncu).

    python tools/prof_dpg.py graph|condense|acoustics
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_00984_b200 import gram_batched  # noqa: E402
from paper_1711_00984_b200.dpg import (acoustics_batched, adjoint_graph_gram_batched,  # noqa: E402
                                       condense_batched)
from paper_1711_00984_b200.inputs import trilinear_batch  # noqa: E402

what = sys.argv[1]
rng = np.random.default_rng(8)
for _ in range(2):
    if what == "graph":
        b = trilinear_batch(512, 21)
        adjoint_graph_gram_batched(4, 2.0, 0.5, b.kind, b.params)
    elif what == "condense":
        bb = trilinear_batch(1024, 22, variable_coef=True)
        G, _ = gram_batched("H1", (5, 5, 5), bb.kind, bb.params, bb.coef)
        B = rng.standard_normal((1024, 216, 125))
        condense_batched(G, B, rng.standard_normal((1024, 216)))
    else:
        b = trilinear_batch(2048, 23)
        acoustics_batched(3, 5, 1.5, b.kind, b.params, rng.uniform(0.5, 1.5, (2048, 216)), parts=False)
torch.cuda.synchronize()
print("ok", what)
