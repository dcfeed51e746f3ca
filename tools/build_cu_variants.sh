#!/bin/bash
# Experiment builds of one kernel file: first argument the .cu file name under
# csrc/, then "tag:nvcc flags" per variant, e.g.
#   bash tools/build_cu_variants.sh sketch_ops.cu "r4:-DRS_SS_RPL=4" "kq4:-DRS_SS_KQ=4"
# -> tools/librskel_<stem>_<tag>.so (load with RSKEL_LIB=... in the tools that honour it).
set -e
SRC=$1; shift
STEM=${SRC%.cu}
cd "$(dirname "$0")/../paper_2310_09417_b200/csrc"
T=$(mktemp -d)
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I ../../include"
for f in *.cu; do [ "$f" = "$SRC" ] || nvcc $F -c $f -o $T/$f.o & done
for v in "$@"; do tag=${v%%:*}; fl=${v#*:}; nvcc $F $fl -c $SRC -o $T/v_$tag.o & done; wait
for v in "$@"; do tag=${v%%:*}; nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/librskel_${STEM}_$tag.so $(ls $T/*.cu.o) $T/v_$tag.o -lcufft; done
rm -rf $T
