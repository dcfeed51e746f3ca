# per-column panel time for experiment builds tools/librskel_exp<bits>.so
for e in ${EXPS:-1 2 4 7}; do echo "== exp $e"; PYTHONPATH=. python tools/panel_nolate.py librskel_exp$e.so 2>&1 | grep "panel R=  2000\|panel R= 20000"; done
