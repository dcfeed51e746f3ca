set -e
export PYTHONPATH=.
python tools/prof_targets.py rank_update > gpurun_out/plain_ru.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rank_update -s 1 -c 1 -o gpurun_out/prof_ru python tools/prof_targets.py rank_update > gpurun_out/ncu_ru.log 2>&1
echo done
