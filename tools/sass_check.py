"""SASS audit of the shipped sm_100a kernels (cuobjdump -sass of the built
library).  Per kernel: FP64 tensor-core MMAs (DMMA), DMMA whose destination
registers overlap an A / B source register, TMA-engine bulk copies (UBLKCP),
and local-memory traffic (LDL / STL = register spills).

    python tools/sass_check.py [--lib PATH] [--out profiles/sass_check_r02.txt]

`check()` is called by __graft_entry__.build(): every specialized general-map
kernel must issue DMMA (the tensor path), and every warp-unit kernel with a
bulk-copy write-out (general_v3, p >= 3) must issue UBLKCP -- a build that
silently lost either fails loudly.  Register overlap D/A, D/B is reported,
not rejected: ptxas emits it in kernels that are verified bit-for-bit against
the oracle, so the hardware reads DMMA sources before writing the
destination (profiles/sass_check_r02.txt)."""

import argparse
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1711_00984_b200", "_lib", "libhexgram_b200.so")

_DMMA = re.compile(r"DMMA\.8x8x4\S*\s+R(\d+)(?:\.\w+)*,\s*R(\d+)(?:\.\w+)*,\s*R(\d+)(?:\.\w+)*,")


def audit(lib=LIB):
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    st = defaultdict(lambda: {"dmma": 0, "d_over_a": 0, "d_over_b": 0, "ublkcp": 0, "local": 0})
    fn = None
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :", 1)[1].strip()
            continue
        if fn is None:
            continue
        s = st[fn]
        if "DMMA" in line:
            m = _DMMA.search(line)
            s["dmma"] += 1
            if m:
                d, a, b = (int(x) for x in m.groups())
                D = set(range(d, d + 4))
                s["d_over_a"] += bool(D & {a, a + 1})
                s["d_over_b"] += bool(D & {b, b + 1})
        elif "UBLKCP" in line:
            s["ublkcp"] += 1
        elif re.search(r"\b(LDL|STL)\b", line):
            s["local"] += 1
    return dict(st)


def _demangle_kernel(name):
    m = re.match(r"_ZN3hxg(\d+)(\w+?)ILi(\d+)ELi(\d+)(?:ELi(\d+))?EE", name)
    if not m:
        return name
    n = int(m.group(1))
    base = m.group(2)[:n]
    args = [g for g in m.groups()[2:] if g is not None]
    return f"{base}<{','.join(args)}>"


def check(lib=LIB):
    st = audit(lib)
    errs = []
    for fn, s in st.items():
        k = _demangle_kernel(fn)
        if k.startswith("general_v3_kernel") or k.startswith("general_v2_kernel"):
            p = int(k.split("<")[1].split(",")[1])
            if p >= 3 and s["dmma"] == 0:
                errs.append(f"{k}: no DMMA")
            if k.startswith("general_v3_kernel") and p >= 3 and s["ublkcp"] == 0:
                errs.append(f"{k}: no UBLKCP (bulk-copy write-out)")
    if errs:
        raise RuntimeError("SASS audit failed: " + "; ".join(errs))
    return st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=LIB)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    st = check(a.lib)
    rows = sorted((_demangle_kernel(f), s) for f, s in st.items() if s["dmma"] or s["ublkcp"] or s["local"])
    tot = defaultdict(int)
    out = ["# SASS audit (cuobjdump -sass of libhexgram_b200.so, sm_100a)",
           "# kernel | DMMA | DMMA with D overlapping A | D overlapping B | UBLKCP | LDL/STL"]
    for k, s in rows:
        out.append(f"{k} | {s['dmma']} | {s['d_over_a']} | {s['d_over_b']} | {s['ublkcp']} | {s['local']}")
        for key in s:
            tot[key] += s[key]
    out.append(f"TOTAL | {tot['dmma']} | {tot['d_over_a']} | {tot['d_over_b']} | {tot['ublkcp']} | {tot['local']}")
    text = "\n".join(out) + "\n"
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
