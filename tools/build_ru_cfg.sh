#!/bin/bash
# Experiment builds of the rank-update streaming kernel's tile configs (RS_RU_VARIANT = 1, 2):
# tools/librskel_ru<N>.so for tools/ru_prof.py (RU_LIB=...).
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = rank_update.cu ] || nvcc $F -c $f -o $T/$f.o & done
for i in ${RU_VARIANTS:-1 2}; do nvcc $F -DRS_RU_VARIANT=$i -c rank_update.cu -o $T/r$i.o & done; wait
for i in ${RU_VARIANTS:-1 2}; do nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_ru$i.so $(ls $T/*.cu.o) $T/r$i.o -lcufft; done
rm -rf $T
