"""Summarise an ncu report: key SOL metrics, instruction mix, stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "--page", "raw")
    h, u, v = rows[0], rows[1], rows[2]
    raw = dict(zip(h, v))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed.sum", "smsp__inst_executed.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed_pipe_fp64.sum", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
    units = dict(zip(h, u))
    summ = {k: (raw.get(k), units.get(k)) for k in keys if k in raw}
    for k, (val, un) in summ.items():
        print(f"{k:70s} {val} {un}")
    sass = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hh = sass[1]
    idx = {k: i for i, k in enumerate(hh)}
    cnt = collections.Counter()
    stalls = collections.Counter()
    scols = [k for k in hh if k.startswith("stall_") and "Not Issued" not in k]
    tot = 0
    for r in sass[2:]:
        if len(r) < len(hh):
            continue
        op = r[idx["Source"]].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        o = o.split(".")[0]
        n = int(r[idx["Instructions Executed"]] or 0)
        cnt[o] += n
        tot += n
        for k in scols:
            try:
                stalls[k] += int(r[idx[k]] or 0)
            except ValueError:
                pass
    print("warp instructions", tot)
    print("mix:", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in cnt.most_common(16)))
    st = sum(stalls.values())
    print("stalls:", ", ".join(f"{k[6:]} {n / st * 100:.1f}%" for k, n in stalls.most_common(10)))
    if len(sys.argv) > 3 and sys.argv[2] == "--json":
        with open(sys.argv[3], "w") as fh:
            json.dump({"metrics": {k: v for k, (v, _) in summ.items()}, "warp_instructions": tot,
                       "mix": dict(cnt.most_common(24)),
                       "stalls": dict(stalls.most_common(12))}, fh, indent=1)


if __name__ == "__main__":
    main()
