#!/bin/bash
# PW kernel: parity (p >= 8 default route, p 4..10 with HXG_PW=1) + p 8..10 timings + optional ncu
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q -x -k "high_order_general or sweep_high_order" 2>&1 | tail -1
HXG_PW=1 python -m pytest tests -m gpu -q -x -k "high_order_general or config_parity_protocol" 2>&1 | tail -1
for p in ${PS:-8 9 10}; do for s in ${SS:-hdiv hcurl h1}; do
  ELEM=${ELEM:-256} bash tools/wl_quick.sh c5_${s}_p${p}_general
done; done
[ -n "$NCU" ] && WLS="$NCU" ELEM=128 bash tools/ncu_pw.sh
true
