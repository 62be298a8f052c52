#!/bin/bash
# PW kernel check: parity at p >= 8 (default route) and at p 4..10 (HXG_PW=1), then timing
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -x -k "high_order_general or sweep_high_order or specialized_equals_generic" 2>&1 | tail -3
HXG_PW=1 python -m pytest tests -m gpu -q -x -k "high_order_general or sweep_high_order or specialized_equals_generic or config_parity_protocol" 2>&1 | tail -3
for p in 8 9 10; do for s in hdiv hcurl h1; do
  ELEM=${ELEM:-256} bash tools/wl_quick.sh c5_${s}_p${p}_general
done; done
for p in 5 6 7; do for s in hdiv hcurl h1; do
  HXG_PW=1 ELEM=${ELEM:-256} bash tools/wl_quick.sh c5_${s}_p${p}_general
done; done
