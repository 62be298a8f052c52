#!/bin/bash
# extrusion kernel: shared-memory budget (trial digits per stage-B pass) sweep
cd "$(dirname "$0")/.."
for kb in ${KBS:-16 40 80}; do echo "ext_smem_kb=$kb"; HXG_EXT_SMEM_KB=$kb tools/wl_quick.sh "$@"; done
