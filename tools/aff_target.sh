#!/bin/bash
cd "$(dirname "$0")/.."
for t in ${TGTS:-256 1024 4096}; do echo "target_kb=$t"; HXG_AFF_TARGET_KB=$t tools/wl_quick.sh "$@"; done
