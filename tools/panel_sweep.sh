#!/bin/bash
for rp in 48 64 96 128 160 224 320 430; do
  echo "rows_per_cta=$rp"
  RSKEL_PANEL_ROWS_PER_CTA=$rp PYTHONPATH=. python tools/bench_kernels.py panel 2>&1 | grep -E "R=  6000|R= 20000"
done
