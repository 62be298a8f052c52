#!/bin/bash
# condensation kernel A/B: warps per CTA (tile = 8 x warps rows)
cd "$(dirname "$0")/.."
for v in "" "-DHXG_CD_WARPS=4"; do
  make -s -B -j16 -C paper_1711_00984_b200/csrc EXTRA="$v" > /dev/null 2>&1 || { echo build fail; continue; }
  echo "EXTRA=$v"; python -m pytest tests/test_dpg.py tests/test_gpu_property.py -q -m gpu -x -k "condense" 2>&1 | tail -1
  python bench.py --no-cpu --steps 3 --e2e-steps -1 > gpurun_out/cd.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/cd.json'))
for s in d['dpg_suite']: print(s['workload'], round(s['elements_per_s']), round(s['roofline_frac'],3))
"
done
