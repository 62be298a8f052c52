"""Where does a general-map kernel differ from the oracle?  Runs one (space, p) on
the general path with the current routing (HXG_PW / HXG_FORCE_V2 from the
environment), compares every element with the CPU oracle and prints the digit
pattern (j1, j2, j3 | i1, i2, i3, block) of the wrong entries.  Test infrastructure."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def digits(space, p, I):
    """(block, d1, d2, d3) of flat index I (spaces.py:9-17 layout)"""
    if space in ("H1", "L2"):
        n = p + 1 if space == "H1" else p
        return (0, I % n, (I // n) % n, I // (n * n))
    for a in range(3):
        ext = [(p + 1 if d == a else p) if space == "Hdiv" else (p if d == a else p + 1) for d in range(3)]
        sz = ext[0] * ext[1] * ext[2]
        if I < sz:
            return (a, I % ext[0], (I // ext[0]) % ext[1], I // (ext[0] * ext[1]))
        I -= sz


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=4)
    ap.add_argument("--space", default="H1")
    ap.add_argument("--p", type=int, default=7)
    a = ap.parse_args()
    import torch

    from oracle import oracle
    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim, trilinear_batch

    p, space = a.p, a.space
    b = trilinear_batch(a.E, 1234, variable_coef=True)
    g, st = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, rule_order=p + 1)
    torch.cuda.synchronize()
    got = g.cpu().numpy()
    ref = oracle.gram_batched(space, "general", (p, p, p), p + 1, b.kind, b.params, b.coef)
    N = dim(space, (p, p, p))
    iu = np.triu_indices(N)
    out = {"space": space, "p": p, "rel_max": float((np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())}
    bad = np.argwhere(np.abs(got - ref) > 1e-9 * np.abs(ref).max())
    out["bad_entries"] = int(bad.shape[0])
    out["total_entries"] = int(got.size)
    if bad.shape[0]:
        rows, cols = iu[0][bad[:, 1]], iu[1][bad[:, 1]]
        out["nan"] = int(np.isnan(got).sum())
        if True:
            dj = np.array([digits(space, p, int(r)) for r in rows[:4000]])
            di = np.array([digits(space, p, int(c)) for c in cols[:4000]])
            for k, nm in ((1, "j1"), (2, "j2"), (3, "j3")):
                out["bad_" + nm] = sorted(set(int(x) for x in dj[:, k]))
            for k, nm in ((1, "i1"), (2, "i2"), (3, "i3")):
                out["bad_" + nm] = sorted(set(int(x) for x in di[:, k]))
            out["bad_j3i3"] = sorted(set((int(x), int(y)) for x, y in zip(dj[:, 3], di[:, 3])))[:40]
            out["bad_blocks"] = sorted(set((int(x), int(y)) for x, y in zip(dj[:, 0], di[:, 0])))
        out["sample"] = [(int(r), int(c), float(got[e, k]), float(ref[e, k])) for (e, k), r, c in
                         list(zip(bad[:6], rows[:6], cols[:6]))]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
