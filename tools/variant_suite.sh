#!/bin/bash
# GPU A/B of compile-time variants: for each EXTRA flag set, rebuild the library,
# run the GPU parity tests selected by $VTESTS (default: v3/v2 vs generic) and the
# bench suite; summaries go to gpurun_out/variant_<i>.txt
cd "$(dirname "$0")/.."
i=0
for extra in "$@"; do
  i=$((i+1)); out=gpurun_out/variant_$i.txt
  echo "EXTRA=$extra" > $out
  make -s -B -j16 -C paper_1711_00984_b200/csrc EXTRA="$extra" > gpurun_out/variant_${i}_build.log 2>&1 || { echo "build failed" >> $out; continue; }
  [ "$VTESTS" = none ] || python -m pytest tests -m gpu -q -x -k "${VTESTS:-specialized or general}" 2>&1 | tail -1 >> $out
  if [ -n "$WL" ]; then tools/wl_quick.sh $WL >> $out; continue; fi
  python bench.py --no-cpu --steps 5 ${BENCH_ARGS} > gpurun_out/variant_$i.json 2> /dev/null
  python - "$i" >> $out <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/variant_{sys.argv[1]}.json"))
for s in d.get("suite", []):
    print(f'{s["workload"]:22s} {s["elements_per_s"]:12.0f} el/s  roof {s["roofline_frac"]:.3f}')
PY
done
cat gpurun_out/variant_*.txt
