#!/bin/bash
# GPU quick check: parity suite + bench suite summary (used during development)
python -m pytest tests -m gpu -q -x 2>&1 | tail -1 > gpurun_out/tests_q.txt
python bench.py --no-cpu --steps 5 ${@} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -2 gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_q.json"))
print("value", round(d["value"]), "frac", round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"]))
for s in d.get("suite", []):
    print(f'{s["workload"]:22s} {s["elements_per_s"]:12.0f} el/s  roof {s["roofline_frac"]:.3f}  fp64 {s["fp64_tflops_alg"]:6.2f} TF  hbm {s["hbm_write_gbs"]:7.0f} GB/s')
PY
cat gpurun_out/tests_q.txt
