#!/bin/bash
# GPU quick check of named workloads: one bench line each (no suite, no CPU leg)
cd "$(dirname "$0")/.."
for w in "$@"; do
  python bench.py --no-cpu --no-suite --steps 3 --e2e-steps -1 --workload $w ${ELEM:+--elements $ELEM} 2>gpurun_out/wl_$w.err | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(f'{\"$w\":26s} {d[\"value\"]:12.0f} el/s  roof {d[\"roofline\"][\"frac\"]:.3f}  ms/step {d[\"ms_per_step\"]:.2f} kern {d[\"roofline\"][\"kernel_ms_per_launch\"]:.2f}')"
done
