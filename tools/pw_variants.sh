#!/bin/bash
# compare PW write-out builds (HXG_LIB variants) on chosen workloads
cd "$(dirname "$0")/.."
HXG_PW=1 python -m pytest tests -m gpu -q -x -k "high_order_general or config_parity_protocol" 2>&1 | grep -E "^FAILED|Error|assert|rel" | head -8
for v in _lib _lib_wb _lib_wo0; do
  echo "== $v"
  for w in ${WL:-c5_hdiv_p8_general c5_hdiv_p10_general c5_hcurl_p10_general}; do
    HXG_LIB=$PWD/paper_1711_00984_b200/$v/libhexgram_b200.so ELEM=${ELEM:-256} bash tools/wl_quick.sh $w
  done
done
