#!/bin/bash
# Experiment build: librskel.so with PANEL_DBG=1 (per-phase clock64 totals printed by the panel
# kernel) -> tools/librskel_paneldbg.so for tools/panel_time.py.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = panel.cu ] || nvcc $F -c $f -o $T/$f.o & done
nvcc $F -DPANEL_DBG=1 $PANEL_EXTRA -c panel.cu -o $T/pdbg.o & wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_paneldbg${PANEL_TAG}.so $(ls $T/*.cu.o) $T/pdbg.o -lcufft
rm -rf $T
