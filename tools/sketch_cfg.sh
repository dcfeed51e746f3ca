# sketch GEMM TF/s for (RSKEL_GEMM_CFG, RSKEL_SK_OVERSUB) pairs
for c in 8 9 12; do for o in 1 2 4; do
  echo -n "cfg $c oversub $o: "; RSKEL_GEMM_CFG=$c RSKEL_SK_OVERSUB=$o PYTHONPATH=. python tools/sketch_width.py 2>&1 | grep "blocks  1 " ; done; done
