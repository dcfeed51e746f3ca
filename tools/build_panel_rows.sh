#!/bin/bash
# Experiment builds of librskel.so with RS_PANEL_ROWS = 192 / 256 / 384 rows per panel CTA:
# tools/librskel_panel{192,256,384}.so for tools/panel_time.py.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = panel.cu ] || nvcc $F -c $f -o $T/$f.o & done
for r in 192 256 384; do nvcc $F -DRS_PANEL_ROWS=$r -c panel.cu -o $T/p$r.o & done; wait
for r in 192 256 384; do nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_panel$r.so $(ls $T/*.cu.o) $T/p$r.o; done
rm -rf $T
