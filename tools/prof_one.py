"""Run the device hot path of one workload a few times (for ncu / compute-sanitizer).

    python tools/prof_one.py c3_hcurl_p6_general [--elements 512] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import DeviceStep  # noqa: E402
from paper_1711_00984_b200.inputs import ALL_WORKLOADS as WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--elements", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
wl = WORKLOADS[a.workload]
dev = torch.device("cuda", 0)
ds = DeviceStep(wl, a.elements or wl.E, 0, dev)
st = torch.cuda.current_stream(dev)
for _ in range(a.reps):
    ev = torch.cuda.Event()
    ds.step(st, ev)
torch.cuda.synchronize()
assert int(ds.status.abs().sum()) == 0
print("ok", a.workload, ds.E)
