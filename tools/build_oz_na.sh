#!/bin/bash
# Experiment builds of librskel.so with OZ_NA_STAGES = A-plane shared-memory stages ($@, e.g. 3 4 6);
# extra nvcc flags in $OZ_EXTRA. Output tools/librskel_ozna<N>.so, loaded by tools/oz_prof.py via OZ_LIB.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = ozaki.cu ] || nvcc $F -c $f -o $T/$f.o & done; wait
for d in "$@"; do nvcc $F $OZ_EXTRA -DOZ_NA_STAGES=$d -c ozaki.cu -o $T/oz$d.o; nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_ozna$d.so $(ls $T/*.cu.o) $T/oz$d.o -lcufft; done
rm -rf $T
