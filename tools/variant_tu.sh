#!/bin/bash
# build a variant library that differs from the in-tree build only in one
# translation unit compiled with extra flags:  tools/variant_tu.sh NAME TU "FLAGS"
# -> paper_1711_00984_b200/_lib_NAME/libhexgram_b200.so (use with HXG_LIB=...)
set -e
cd "$(dirname "$0")/../paper_1711_00984_b200"
d=_lib_$1
mkdir -p $d/obj
cp _lib/obj/*.o $d/obj/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
     --expt-relaxed-constexpr $3 -c -o $d/obj/$2.o csrc/$2.cu > $d/obj/$2.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libhexgram_b200.so $d/obj/*.o
echo "built $d"
