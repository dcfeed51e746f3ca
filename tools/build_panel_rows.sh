#!/bin/bash
# Experiment builds of librskel.so: panel rows per CTA (RS_PANEL_ROWS) and smallest polling
# width (RS_PANEL_QMIN): tools/librskel_panel_<rows>_<qmin>.so for tools/panel_time.py.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
V="128_2 128_3 64_0 64_2 96_2"
for f in *.cu; do [ "$f" = panel.cu ] || nvcc $F -c $f -o $T/$f.o & done
for v in $V; do r=${v%_*}; q=${v#*_}; nvcc $F -DRS_PANEL_ROWS=$r -DRS_PANEL_QMIN=$q -c panel.cu -o $T/p$v.o & done; wait
for v in $V; do nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_panel_$v.so $(ls $T/*.cu.o) $T/p$v.o; done
rm -rf $T
