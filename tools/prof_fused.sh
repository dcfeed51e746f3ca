set -e
export PYTHONPATH=.
python tools/prof_targets.py fused 3 > gpurun_out/plain_fused.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_absorb -s 1 -c 1 -o gpurun_out/prof_fused python tools/prof_targets.py fused 3 > gpurun_out/ncu_fused.log 2>&1
echo done
