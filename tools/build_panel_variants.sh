#!/bin/bash
# Experiment builds of the panel: each argument is "tag:nvcc flags", e.g.
#   bash tools/build_panel_variants.sh "flat:-DRS_PANEL_CLUSTER=1" "b64:-DRS_PANEL_CLUSTER=1 -DRS_PANEL_BACKOFF=64"
# -> tools/librskel_panel_<tag>.so for tools/panel_time.py.
set -e
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = panel.cu ] || nvcc $F -c $f -o $T/$f.o & done
for v in "$@"; do tag=${v%%:*}; fl=${v#*:}; nvcc $F $fl -c panel.cu -o $T/p_$tag.o & done; wait
for v in "$@"; do tag=${v%%:*}; nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_panel_$tag.so $(ls $T/*.cu.o) $T/p_$tag.o -lcufft; done
rm -rf $T
