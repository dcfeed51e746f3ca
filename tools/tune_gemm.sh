#!/bin/bash
# Compare GEMM tile configurations (RSKEL_GEMM_CFG) on the skeleton shapes.
for c in ${CFGS:-0 8 12}; do
  echo "=== cfg $c"
  RSKEL_GEMM_CFG=$c PYTHONPATH=. python tools/bench_kernels.py gemm 2>&1 | grep -E "sketch gemm|schur k|err"
done
