set -e
export PYTHONPATH=.
python tools/prof_targets.py panel > gpurun_out/plain_panel.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 1 -c 1 -o gpurun_out/prof_panel python tools/prof_targets.py panel > gpurun_out/ncu_panel.log 2>&1
echo done
