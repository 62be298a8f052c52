"""Investigation harness for general_v3_kernel<H1, 7, 8> (round-1 "known
compiler issue"): run H1 p = 7 on the general path with the v3 kernel
(HXG_V3_P7=1) and with the v2 kernel, compare both against the CPU oracle,
and print where the v3 result differs (rows / columns / units).

Used under compute-sanitizer (racecheck / synccheck / initcheck / memcheck)
by tools/v3p7_check.sh.  Test infrastructure only."""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--space", default="H1")
    ap.add_argument("--p", type=int, default=7)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    import torch

    from paper_1711_00984_b200 import gram_batched
    from paper_1711_00984_b200.inputs import dim, trilinear_batch

    p, space = args.p, args.space
    b = trilinear_batch(args.E, 1234, variable_coef=True)
    res = {}
    for name, env in (("v3", "1"), ("v2", None)):
        if env is None:
            os.environ.pop("HXG_V3_P7", None)
            os.environ["HXG_FORCE_V2"] = "1"
        else:
            os.environ["HXG_V3_P7"] = env
            os.environ.pop("HXG_FORCE_V2", None)
        g, st = gram_batched(space, (p, p, p), b.kind, b.params, b.coef, rule_order=p + 1)
        torch.cuda.synchronize()
        res[name] = g.cpu().numpy()
    os.environ.pop("HXG_FORCE_V2", None)
    os.environ.pop("HXG_V3_P7", None)
    N = dim(space, (p, p, p))
    out = {"space": space, "p": p, "E": args.E}
    d = np.abs(res["v3"] - res["v2"])
    rel = np.linalg.norm(res["v3"] - res["v2"], axis=1) / np.linalg.norm(res["v2"], axis=1)
    out["v3_vs_v2_rel_max"] = float(rel.max())
    bad = np.argwhere(d > 1e-10 * np.abs(res["v2"]).max())
    out["bad_entries"] = int(bad.shape[0])
    if bad.shape[0]:
        iu = np.triu_indices(N)
        rows, cols = iu[0][bad[:, 1]], iu[1][bad[:, 1]]
        out["bad_elements"] = sorted(set(int(x) for x in bad[:, 0]))[:16]
        out["bad_rows_first"] = sorted(set(int(x) for x in rows))[:32]
        out["bad_cols_first"] = sorted(set(int(x) for x in cols))[:32]
        n1 = p + 1
        out["bad_j3_i3"] = sorted(set((int(r) // (n1 * n1), int(c) // (n1 * n1)) for r, c in zip(rows, cols)))[:32]
    if not args.no_oracle:
        from oracle import oracle

        ref = oracle.gram_batched(space, "general", (p, p, p), p + 1, b.kind, b.params, b.coef)
        for name in ("v3", "v2"):
            r = np.linalg.norm(res[name] - ref, axis=1) / np.linalg.norm(ref, axis=1)
            out[f"{name}_vs_oracle_rel_max"] = float(r.max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
