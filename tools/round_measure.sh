#!/bin/bash
# One GPU call that refreshes every committed measurement of the round (gpurun_out/ -> profiles/):
#   tests, the bench line, the reference arm, determinism at full size, the step launch list,
#   the ncu capture of the sketch kernel, the secondary configs, and the N > 1 bench plumbing
#   (gloo, 2 ranks sharing the GPU, cfg5 recipe at 16384).
cd "$(dirname "$0")/.."
O=gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/m_gputest.log 2>&1; echo "rc=$?" >> $O/m_gputest.log
python bench.py --steps 3 --warmup 3 > $O/m_bench.log 2>&1
python bench.py --impl reference --steps 1 --warmup 1 > $O/m_bench_ref.log 2>&1
python tools/determinism_full.py --cfg 2 --host > $O/m_det_cfg2.jsonl 2>&1
python tools/determinism_full.py --cfg 5 > $O/m_det_cfg5.jsonl 2>&1
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/m_step_launches.csv python tools/prof_step.py > $O/m_prof_step.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:oz_gemm -c 1 -s 2 -o $O/m_oz_gemm \
    python tools/oz_prof.py > $O/m_oz_prof.log 2>&1
python bench_configs.py cfg1 cfg3 cfg4 cfg5 > $O/m_configs.jsonl 2>&1
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --size 16384 --e2e-steps 1 --no-cpu \
    > $O/m_bench_n2_gloo.log 2>&1
echo done > $O/m_done
