#!/bin/bash
# Round evaluation on one B200: gpu tests, smoke, bench, ncu launch list, ncu full captures.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python bench_configs.py --cpu > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?" >> gpurun_out/configs.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
KRE='regex:dgemm|panel|rank_update|sumsq|trinv|gather|perm_update|scatter|fixup|iota|transpose|rng_'
python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -s 4000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu \
    > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/ncu_launches.log
ncu --set full --clock-control none --import-source on -k regex:dgemm_kernel -s 40 -c 1 \
    -o gpurun_out/prof_bench_sketch python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full.log
ncu --set full --clock-control none --import-source on -k regex:rank_update -s 100 -c 1 \
    -o gpurun_out/prof_bench_ru python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu \
    > gpurun_out/ncu_full_ru.log 2>&1
echo "full ru rc=$?" >> gpurun_out/ncu_full_ru.log
for r in prof_bench_sketch prof_bench_ru; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
tail -n 3 gpurun_out/*.log
