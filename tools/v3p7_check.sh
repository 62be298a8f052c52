#!/bin/bash
# general_v3_kernel<H1, 7, 8> investigation (GPU box): parity of v3 vs v2 vs the
# oracle on the product build and on the HXG_DMMA_KEEP=1 build, then the four
# compute-sanitizer tools on a small batch.  Output: gpurun_out/v3p7_*.txt
cd "$(dirname "$0")/.."
O=gpurun_out
python tools/v3p7_check.py --E 64 > $O/v3p7_parity.txt 2>&1
HXG_LIB=$PWD/paper_1711_00984_b200/_lib_keep/libhexgram_b200.so python tools/v3p7_check.py --E 64 > $O/v3p7_parity_keep.txt 2>&1
for sp in Hcurl Hdiv; do python tools/v3p7_check.py --E 16 --space $sp >> $O/v3p7_parity_other.txt 2>&1; done
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/v3p7_check.py --E 2 --no-oracle \
    > $O/v3p7_san_$tool.txt 2>&1
  echo "$tool exit $?" >> $O/v3p7_san_summary.txt
  tail -3 $O/v3p7_san_$tool.txt >> $O/v3p7_san_summary.txt
done
cat $O/v3p7_parity.txt $O/v3p7_parity_keep.txt $O/v3p7_parity_other.txt $O/v3p7_san_summary.txt
