#!/bin/bash
# Experiment builds of librskel.so with other row-major DMMA tile configs (RS_ROW_CFG):
# tools/librskel_row{1,2,3}.so for tools/schur_cfg.py.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = gemm_f64.cu ] || nvcc $F -c $f -o $T/$f.o & done; wait
for i in ${ROW_VARIANTS:-1 2 3}; do nvcc $F -DRS_ROW_VARIANT=$i -c gemm_f64.cu -o $T/g$i.o & done; wait
for i in ${ROW_VARIANTS:-1 2 3}; do nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_row$i.so $(ls $T/*.cu.o) $T/g$i.o -lcufft; done
rm -rf $T
