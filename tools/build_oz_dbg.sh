#!/bin/bash
# Experiment builds of librskel.so with OZ_DBG=1 (no MMAs) / 2 (no epilogue TMEM work):
# tools/librskel_ozdbg{1,2}.so, loaded by tools/oz_prof.py via OZ_LIB.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = ozaki.cu ] || nvcc $F -c $f -o $T/$f.o & done; wait
for d in 1 2; do nvcc $F -DOZ_DBG=$d -c ozaki.cu -o $T/oz$d.o; nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_ozdbg$d.so $(ls $T/*.cu.o) $T/oz$d.o; done
rm -rf $T
