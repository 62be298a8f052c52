"""Print the config-5 sweep JSON (bench.py --sweep) as a space x p table of roofline %."""
import json
import sys

d = json.load(open(sys.argv[1]))
rows = {}
for p in d["points"]:
    rows.setdefault((p["space"], p["path"]), {})[p["p_test"]] = p["roofline_frac"]
ps = sorted({p["p_test"] for p in d["points"]})
print("space/path".ljust(18) + "".join(f"{q:>5d}" for q in ps))
for k, v in rows.items():
    print(f"{k[0]}/{k[1]}".ljust(18) + "".join(f"{100 * v[q]:5.0f}" if q in v else "    -" for q in ps))
