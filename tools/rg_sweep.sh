#!/bin/bash
# affine kernel: row groups per CTA (HXG_AFF_RG) sweep over workloads
cd "$(dirname "$0")/.."
for rg in ${RGS:-1 2 4 8 100}; do
  echo "rg=$rg"
  HXG_AFF_RG=$rg tools/wl_quick.sh "$@"
done
